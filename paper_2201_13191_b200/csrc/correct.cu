// correct.cu — the correction loop's elementwise stages around the projector
// (SURVEY.md §8(f) rank 1): REF intensity_to_attenuation (recon.cpp:324-348),
// correct_projections / Eq. 8 (correction.cpp:58-86) and the loop's tail after
// the Monte Carlo runs (correction.cpp:199-246).
//
// The tail is fused: the scatter stack's column up-sampling pass (the last
// Catmull-Rom pass, REF postprocess.cpp:235-252) computes each full-resolution
// scatter pixel in registers and applies the primary floor, the scatter-
// fraction statistic and Eq. 8 right there; the primary's column pass runs
// twice (once for each view's peak, once inside the correction), so neither
// up-sampled stack (720 x 2048^2 x 8 B = 24 GB each in REF's C5 loop) is
// ever written.
//
// Counts (clamped negative scatter, bad pixels) are integers and the mean
// scatter fraction is summed as 2 x 32-bit fixed-point limbs per pixel, so
// every statistic is independent of the thread schedule.
#include <cstdint>

#include "xs_types.h"

namespace xsd {

struct CorrectStats {
    unsigned long long clamped;   // negative scatter pixels clamped to 0
    unsigned long long bad;       // non-positive primary / intensity / flat-field pixels
    unsigned long long frac_hi;   // sum of floor(f * 2^32)
    unsigned long long frac_lo;   // sum of the next 32 bits of f
    unsigned long long frac_n;    // pixels with Ip + Is > 0
    unsigned long long peak[1];   // per-view primary peak (bits of a non-negative double), n_views
};

namespace {

__device__ __forceinline__ unsigned long long warp_sum(unsigned long long v)
{
#pragma unroll
    for (int o = 16; o; o >>= 1)
        v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// one atomic per warp for each counter
__device__ __forceinline__ void add_stats(CorrectStats* st, unsigned long long clamped, unsigned long long bad,
                                          unsigned long long fh, unsigned long long fl, unsigned long long fn)
{
    clamped = warp_sum(clamped);
    bad = warp_sum(bad);
    fh = warp_sum(fh);
    fl = warp_sum(fl);
    fn = warp_sum(fn);
    if ((threadIdx.x & 31) == 0) {
        if (clamped)
            atomicAdd(&st->clamped, clamped);
        if (bad)
            atomicAdd(&st->bad, bad);
        if (fh)
            atomicAdd(&st->frac_hi, fh);
        if (fl)
            atomicAdd(&st->frac_lo, fl);
        if (fn)
            atomicAdd(&st->frac_n, fn);
    }
}

// REF intensity_to_attenuation: a = ln(flat / I) where I > 0; bad pixels
// (also non-positive flat-field pixels, counted once) are counted.
__global__ void i2a_kernel(const double* __restrict__ in, const double* __restrict__ flat,
                           double* __restrict__ out, size_t npix, int n_img, CorrectStats* st)
{
    unsigned long long bad = 0;
    const size_t n = npix * n_img;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t base = (size_t)blockIdx.x * blockDim.x; base < n; base += stride) {
        const size_t i = base + threadIdx.x;
        if (i < n) {
            const size_t p = i % npix;
            const double v = in[i];
            if (i < npix && !(flat[p] > 0.0))
                ++bad;
            if (!(v > 0.0)) {
                ++bad;
                out[i] = 0.0;
            } else {
                out[i] = log(flat[p] / v);
            }
        }
    }
    add_stats(st, 0, bad, 0, 0, 0);
}

// REF correct_projections: c = a - ln(Ip / (Ip + max(Is, 0)))
__device__ __forceinline__ double eq8(double a, double ip, double is, unsigned long long& clamped,
                                      unsigned long long& bad)
{
    if (!(ip > 0.0))
        ++bad;
    if (is < 0.0) {
        is = 0.0;
        ++clamped;
    }
    return a - log(ip / (ip + is));
}

__global__ void correct_kernel(const double* __restrict__ a, const double* __restrict__ ip,
                               const double* __restrict__ is, double* __restrict__ out, size_t n,
                               CorrectStats* st)
{
    unsigned long long clamped = 0, bad = 0;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t base = (size_t)blockIdx.x * blockDim.x; base < n; base += stride) {
        const size_t i = base + threadIdx.x;
        if (i < n)
            out[i] = eq8(a[i], ip[i], is[i], clamped, bad);
    }
    add_stats(st, clamped, bad, 0, 0, 0);
}

// Catmull-Rom sample (REF fetch + catmull_rom_pass, postprocess.cpp:201-233);
// the same arithmetic as postprocess.cu.
__device__ __forceinline__ double cr_fetch_c(const double* line, int n, size_t stride, int i)
{
    if (n == 1)
        return line[0];
    if (i < 0)
        return line[0] + i * (line[stride] - line[0]);
    if (i >= n)
        return line[(size_t)(n - 1) * stride] +
               (i - (n - 1)) * (line[(size_t)(n - 1) * stride] - line[(size_t)(n - 2) * stride]);
    return line[(size_t)i * stride];
}

__device__ __forceinline__ double cr_sample_c(const double* line, int n_in, int n_out, size_t stride, int i)
{
    const double scale = (double)n_in / n_out;
    const double x = (i + 0.5) * scale - 0.5;
    const int base = (int)floor(x);
    const double t = x - base;
    const double t2 = t * t, t3 = t2 * t;
    const double w0 = 0.5 * (-t3 + 2.0 * t2 - t);
    const double w1 = 0.5 * (3.0 * t3 - 5.0 * t2 + 2.0);
    const double w2 = 0.5 * (-3.0 * t3 + 4.0 * t2 + t);
    const double w3 = 0.5 * (t3 - t2);
    return w0 * cr_fetch_c(line, n_in, stride, base - 1) + w1 * cr_fetch_c(line, n_in, stride, base) +
           w2 * cr_fetch_c(line, n_in, stride, base + 1) + w3 * cr_fetch_c(line, n_in, stride, base + 2);
}

// Column passes loop over rows (blockIdx.y strides by gridDim.y) so that the
// statistics are reduced in registers and then once per block: per-warp
// atomics on a handful of addresses would serialise at L2 (94M of them for a
// 720 x 2048^2 stack).
constexpr int kRowGroups = 16; // row chunks per column (contiguous rows: the 4 taps are reused)

__device__ __forceinline__ unsigned long long block_sum(unsigned long long v, unsigned long long* sh)
{
    v = warp_sum(v);
    const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    __syncthreads();
    if ((threadIdx.x & 31) == 0)
        sh[w] = v;
    __syncthreads();
    unsigned long long t = 0;
    for (int i = 0; i < nw; ++i)
        t += sh[i];
    return t;
}

// primary column pass, statistics only: peak[view] = max(0, max of the
// up-sampled view).  The correction pass recomputes the primary pixels in
// registers, so the full-resolution primary stack is never stored either.
__global__ void cr_cols_peak_kernel(const double* __restrict__ tmp, int nu_out, int nv, int nv_out,
                                    CorrectStats* st)
{
    __shared__ double shm[32];
    const int iu = blockIdx.x * blockDim.x + threadIdx.x;
    const int chunk = (nv_out + gridDim.y - 1) / gridDim.y;
    const int j0 = blockIdx.y * chunk, j1 = j0 + chunk < nv_out ? j0 + chunk : nv_out;
    double m = 0.0;
    if (iu < nu_out) {
        const double* line = tmp + (size_t)blockIdx.z * nu_out * nv + iu;
        for (int j = j0; j < j1; ++j) {
            const double v = cr_sample_c(line, nv, nv_out, (size_t)nu_out, j);
            m = v > m ? v : m;
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1)
        m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0)
        shm[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 1; i < (int)(blockDim.x >> 5); ++i)
            m = fmax(m, shm[i]);
        if (m > 0.0) // non-negative doubles order like their bits
            atomicMax(&st->peak[blockIdx.z], (unsigned long long)__double_as_longlong(m));
    }
}

// column passes of both stacks fused with the primary floor, the mean-
// scatter-fraction sums and Eq. 8 (REF correction.cpp:206-246)
__global__ void cr_cols_correct_kernel(const double* __restrict__ tmp_p, const double* __restrict__ tmp_s,
                                       const double* __restrict__ a, double* __restrict__ out, int nu_out,
                                       int nv, int nv_out, CorrectStats* st)
{
    __shared__ unsigned long long sh[32];
    const int iu = blockIdx.x * blockDim.x + threadIdx.x;
    const int chunk = (nv_out + gridDim.y - 1) / gridDim.y;
    const int j0 = blockIdx.y * chunk, j1 = j0 + chunk < nv_out ? j0 + chunk : nv_out;
    unsigned long long clamped = 0, bad = 0, fh = 0, fl = 0, fn = 0;
    if (iu < nu_out) {
        const size_t col = (size_t)blockIdx.z * nu_out * nv + iu;
        const double peak = __longlong_as_double((long long)st->peak[blockIdx.z]);
        const double floor_val = 1e-12 * peak;
        for (int j = j0; j < j1; ++j) {
            const double pv = cr_sample_c(tmp_p + col, nv, nv_out, (size_t)nu_out, j);
            const double s = cr_sample_c(tmp_s + col, nv, nv_out, (size_t)nu_out, j);
            const size_t o = (size_t)blockIdx.z * nu_out * nv_out + (size_t)j * nu_out + iu;
            const double ip = pv > floor_val ? pv : floor_val; // std::max(v, floor_val)
            const double isc = s > 0.0 ? s : 0.0;              // std::max(0.0, s)
            if (ip + isc > 0.0) {
                const double f = isc / (ip + isc); // in [0, 1]
                const double f32 = f * 4294967296.0;
                const double h = floor(f32);
                fh += (unsigned long long)h;
                fl += (unsigned long long)floor((f32 - h) * 4294967296.0);
                ++fn;
            }
            out[o] = eq8(a[o], ip, s, clamped, bad);
        }
    }
    clamped = block_sum(clamped, sh);
    bad = block_sum(bad, sh);
    fh = block_sum(fh, sh);
    fl = block_sum(fl, sh);
    fn = block_sum(fn, sh);
    if (threadIdx.x == 0) {
        if (clamped)
            atomicAdd(&st->clamped, clamped);
        if (bad)
            atomicAdd(&st->bad, bad);
        if (fh)
            atomicAdd(&st->frac_hi, fh);
        if (fl)
            atomicAdd(&st->frac_lo, fl);
        if (fn)
            atomicAdd(&st->frac_n, fn);
    }
}

// rows: in (nv x nu) -> tmp (nv x nu_out)
__global__ void cr_rows_c(const double* __restrict__ in, double* __restrict__ tmp, int nu, int nv, int nu_out)
{
    const int iv = blockIdx.y;
    const double* line = in + (size_t)blockIdx.z * nu * nv + (size_t)iv * nu;
    double* o = tmp + (size_t)blockIdx.z * nu_out * nv + (size_t)iv * nu_out;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nu_out; i += gridDim.x * blockDim.x)
        o[i] = cr_sample_c(line, nu, nu_out, 1, i);
}

} // namespace

size_t correct_stats_bytes(int n_views) { return sizeof(CorrectStats) + (size_t)(n_views > 1 ? n_views - 1 : 0) * 8; }

cudaError_t launch_i2a(const double* in, const double* flat, double* out, size_t npix, int n_img,
                       void* stats, int sm_count, cudaStream_t s)
{
    i2a_kernel<<<sm_count * 8, 256, 0, s>>>(in, flat, out, npix, n_img, static_cast<CorrectStats*>(stats));
    return cudaGetLastError();
}

cudaError_t launch_correct(const double* a, const double* ip, const double* is, double* out, size_t n,
                           void* stats, int sm_count, cudaStream_t s)
{
    correct_kernel<<<sm_count * 8, 256, 0, s>>>(a, ip, is, out, n, static_cast<CorrectStats*>(stats));
    return cudaGetLastError();
}

// in: primary (nv x nu per view) and the angle-interpolated scatter stack at
// the Monte Carlo resolution; tmp: 2 x n_views x nv x nu_out (the row passes)
cudaError_t launch_correction_tail(const double* primary, const double* scatter, const double* a, double* tmp,
                                   double* out, int nu, int nv, int n_views, int nu_out, int nv_out, void* stats,
                                   cudaStream_t s)
{
    CorrectStats* st = static_cast<CorrectStats*>(stats);
    double* tmp_p = tmp;
    double* tmp_s = tmp + (size_t)n_views * nv * nu_out;
    const dim3 rows((nu_out + 127) / 128, nv, n_views),
        cols((nu_out + 127) / 128, nv_out < kRowGroups ? nv_out : kRowGroups, n_views);
    cr_rows_c<<<rows, 128, 0, s>>>(primary, tmp_p, nu, nv, nu_out);
    cr_rows_c<<<rows, 128, 0, s>>>(scatter, tmp_s, nu, nv, nu_out);
    cr_cols_peak_kernel<<<cols, 128, 0, s>>>(tmp_p, nu_out, nv, nv_out, st);
    cr_cols_correct_kernel<<<cols, 128, 0, s>>>(tmp_p, tmp_s, a, out, nu_out, nv, nv_out, st);
    return cudaGetLastError();
}

} // namespace xsd
