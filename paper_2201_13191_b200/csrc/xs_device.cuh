// xs_device.cuh — device-side building blocks of the B200 projector.
//
// Everything that the transport and primary kernels share: the Philox
// stream (REF rng.hpp), table interpolation (REF table.hpp), the voxel
// formats, the exact Siddon walker set-up (REF trace.cpp:22-103), and the
// fixed-point tallies (include/xscat_gpu.h).
//
// Arithmetic follows the reference's expression order and the library is
// compiled with -fmad=false, so every basic operation rounds like the
// reference's x86-64 build; only libm transcendentals (log, exp, sin, cos,
// acos) may differ in the last ulp from glibc.
#pragma once

#include <cstdint>

#include "../../include/xscat_gpu.h"
#include "xs_types.h"

namespace xsd {

constexpr double kPi = 3.14159265358979323846;
constexpr double kR0 = 2.8179403e-13;  // constants.hpp:9
constexpr double kMec2 = 511.0;        // constants.hpp:12
constexpr double kHc = 12.398;         // constants.hpp:15
constexpr double kBarn = 1.0e-24;      // constants.hpp:18

// ------------------------------------------------------------------ errors
// First error wins; the host maps code -> xs_status and formats REF's message.
__device__ __forceinline__ void raise(DevStatus* st, int code, int what, int bin, double e,
                                      double v)
{
    if (atomicCAS(&st->code, 0, code) == 0) {
        st->what = what;
        st->bin = bin;
        st->energy = e;
        st->value = v;
    }
}

// ------------------------------------------------------------------- Philox
// REF rng.hpp:11-67; key = seed, counter = {block, photon, bin, angle}.
struct Rng {
    uint32_t photon, bin, block, pos;
    uint32_t b0, b1, b2, b3;
};

__device__ __forceinline__ void rng_init(Rng& r, uint32_t photon, uint32_t bin)
{
    r.photon = photon;
    r.bin = bin;
    r.block = 0;
    r.pos = 4;
}

__device__ __forceinline__ void rng_refill(Rng& r, uint32_t k0, uint32_t k1, uint32_t angle)
{
    uint32_t c0 = r.block, c1 = r.photon, c2 = r.bin, c3 = angle;
#pragma unroll
    for (int i = 0; i < 10; ++i) {
        const uint32_t lo0 = 0xD2511F53u * c0, hi0 = __umulhi(0xD2511F53u, c0);
        const uint32_t lo1 = 0xCD9E8D57u * c2, hi1 = __umulhi(0xCD9E8D57u, c2);
        c0 = hi1 ^ c1 ^ k0;
        c1 = lo1;
        c2 = hi0 ^ c3 ^ k1;
        c3 = lo0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    r.b0 = c0;
    r.b1 = c1;
    r.b2 = c2;
    r.b3 = c3;
    r.pos = 0;
    ++r.block;
}

// uniform() consumes two u32 (rng.hpp:29-35); every draw of the transport
// is a uniform(), so pos is always 0, 2 or 4.
__device__ __forceinline__ double rng_uniform(Rng& r, uint32_t k0, uint32_t k1, uint32_t angle)
{
    if (r.pos == 4)
        rng_refill(r, k0, k1, angle);
    uint64_t hi, lo;
    if (r.pos == 0) {
        hi = r.b0;
        lo = r.b1;
    } else {
        hi = r.b2;
        lo = r.b3;
    }
    r.pos += 2;
    const uint64_t bits = ((hi << 32) | lo) >> 11;
    return ((double)bits + 0.5) * 0x1p-53;
}

// ------------------------------------------------------------------- tables
// Packed table: x[n], y[n], lx[n] = log x, ly[n] = log y (host glibc logs).
struct Tab {
    const double* x;
    const double* y;
    const double* lx;
    const double* ly;
    int n;
};

__device__ __forceinline__ Tab tab_at(const double* base, TabDesc d)
{
    Tab t;
    t.x = base + d.off;
    t.y = t.x + d.n;
    t.lx = t.y + d.n;
    t.ly = t.lx + d.n;
    t.n = d.n;
    return t;
}

// REF table.hpp:73-91; returns false when out of range.
__device__ __forceinline__ bool tab_locate(const Tab& t, double x, int& idx, bool& exact)
{
    const double x0 = __ldg(t.x), xn = __ldg(t.x + t.n - 1);
    if (!(x >= x0 && x <= xn))
        return false;
    int lo = 0, hi = t.n - 1;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (__ldg(t.x + mid) <= x)
            lo = mid;
        else
            hi = mid;
    }
    if (x == __ldg(t.x + lo)) {
        idx = lo;
        exact = true;
    } else if (x == __ldg(t.x + hi)) {
        idx = hi;
        exact = true;
    } else {
        idx = lo;
        exact = false;
    }
    return true;
}

__device__ __forceinline__ bool tab_linear(const Tab& t, double x, double& y)
{
    int i;
    bool ex;
    if (!tab_locate(t, x, i, ex))
        return false;
    if (ex) {
        y = __ldg(t.y + i);
        return true;
    }
    const double x0 = __ldg(t.x + i), x1 = __ldg(t.x + i + 1);
    const double y0 = __ldg(t.y + i), y1 = __ldg(t.y + i + 1);
    const double u = (x - x0) / (x1 - x0);
    y = y0 + u * (y1 - y0);
    return true;
}

__device__ __forceinline__ double tab_linear_clamped(const Tab& t, double x)
{
    if (x <= __ldg(t.x))
        return __ldg(t.y);
    if (x >= __ldg(t.x + t.n - 1))
        return __ldg(t.y + t.n - 1);
    double y = 0.0;
    tab_linear(t, x, y);
    return y;
}

// REF table.hpp:57-69 with the knot logarithms precomputed on the host.
__device__ __forceinline__ bool tab_loglog(const Tab& t, double x, double& y)
{
    int i;
    bool ex;
    if (!tab_locate(t, x, i, ex))
        return false;
    if (ex) {
        y = __ldg(t.y + i);
        return true;
    }
    const double y0 = __ldg(t.y + i), y1 = __ldg(t.y + i + 1);
    if (y0 <= 0.0 || y1 <= 0.0) {
        const double x0 = __ldg(t.x + i), x1 = __ldg(t.x + i + 1);
        const double u = (x - x0) / (x1 - x0);
        y = y0 + u * (y1 - y0);
        return true;
    }
    const double lx0 = __ldg(t.lx + i), lx1 = __ldg(t.lx + i + 1);
    const double ly0 = __ldg(t.ly + i), ly1 = __ldg(t.ly + i + 1);
    const double u = (log(x) - lx0) / (lx1 - lx0);
    y = exp(ly0 + u * (ly1 - ly0));
    return true;
}

// ------------------------------------------------------------ voxel formats
// 4x4x4 bricks; bricks x-fastest.  P4: 32 B / brick (nibbles), P8 and raw
// ids: 64 B / brick, raw density: 256 B / brick.
__device__ __forceinline__ uint32_t brick_cell(const Grid& G, int ix, int iy, int iz)
{
    const uint32_t brick = (uint32_t)(ix >> 2) +
                           (uint32_t)G.nbx * ((uint32_t)(iy >> 2) + (uint32_t)G.nby * (uint32_t)(iz >> 2));
    const uint32_t within = (uint32_t)(ix & 3) | ((uint32_t)(iy & 3) << 2) | ((uint32_t)(iz & 3) << 4);
    return (brick << 6) | within;
}

__device__ __forceinline__ int load_code_p4(const Grid& G, uint32_t c)
{
    const uint8_t b = __ldg(G.vox + (c >> 1));
    return (b >> ((c & 1u) << 2)) & 0xF;
}

__device__ __forceinline__ int load_code_p8(const Grid& G, uint32_t c) { return __ldg(G.vox + c); }

__device__ __forceinline__ float load_density_raw(const Grid& G, uint32_t c)
{
    return __ldg(G.dens + c);
}

// Half-open voxel index (REF trace.cpp:60-64).
__device__ __forceinline__ int voxel_of(double p, double org, double inv_h, int n)
{
    int i = (int)floor((p - org) * inv_h);
    return i < 0 ? 0 : (i > n - 1 ? n - 1 : i);
}

// ------------------------------------------------------- fixed-point tallies
// include/xscat_gpu.h xs_quantize; q = x / 2^log2_unit.
__device__ __forceinline__ bool quantize(double q, uint64_t& l0, uint64_t& l1, uint64_t& l2)
{
    if (!(q >= 0.0) || !(q < 4294967296.0))
        return false;
    const double i2 = floor(q);
    const double r1 = (q - i2) * 4294967296.0;
    const double i1 = floor(r1);
    const double r2 = (r1 - i1) * 4294967296.0;
    l2 = (uint64_t)i2;
    l1 = (uint64_t)i1;
    l0 = (uint64_t)rint(r2);
    return true;
}

__device__ __forceinline__ void red_add(unsigned long long* p, uint64_t v)
{
    if (v)
        atomicAdd(p, (unsigned long long)v);
}

__device__ __forceinline__ bool tally_global(unsigned long long* slot, double x, int log2_unit)
{
    uint64_t l0, l1, l2;
    if (!quantize(ldexp(x, -log2_unit), l0, l1, l2))
        return false;
    red_add(slot + 0, l0);
    red_add(slot + 1, l1);
    red_add(slot + 2, l2);
    return true;
}

// include/xscat_gpu.h xs_dequantize, same operation sequence.
__device__ __forceinline__ double dequantize(uint64_t s0, uint64_t s1, uint64_t s2, int log2_unit)
{
    uint64_t lo = s0;
    uint64_t hi = s2;
    const uint64_t t = s1 << 32;
    const uint64_t c = s1 >> 32;
    const uint64_t lo2 = lo + t;
    hi += c + (lo2 < lo ? 1u : 0u);
    lo = lo2;
    return ldexp((double)hi * 18446744073709551616.0 + (double)lo, log2_unit - 64);
}

} // namespace xsd
