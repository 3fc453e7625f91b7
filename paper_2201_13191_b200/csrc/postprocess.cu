// postprocess.cu — scatter post-processing stencils of the correction loop
// (REF postprocess.cpp; call order in correction.cpp:199-224).
//
// All kernels are batched over a stack of images (blockIdx.z = image) and
// keep the reference's fp64 arithmetic and summation order, so results are
// bit-identical to the reference (tests/test_postprocess_gpu.py).  They are
// HBM-streaming stencils: one coalesced read pass and one write pass per
// separable direction.
#include <cstdint>

#include "xs_types.h"

namespace xsd {

// ---------------------------------------------------------- Savitzky-Golay
// REF sg_pass (postprocess.cpp:106-122).  K holds the (half+1)^2 truncated
// kernels, kernel (left, right) at K + (left*(half+1)+right)*W, W = 2*half+1.
__global__ void sg_rows_kernel(const double* __restrict__ in, double* __restrict__ out, int nu,
                               int nv, int half, const double* __restrict__ K)
{
    const int W = 2 * half + 1;
    const int iv = blockIdx.y;
    const size_t img = (size_t)blockIdx.z * nu * nv;
    const double* row = in + img + (size_t)iv * nu;
    double* orow = out + img + (size_t)iv * nu;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nu; i += gridDim.x * blockDim.x) {
        const int left = i < half ? i : half;
        const int right = (nu - 1 - i) < half ? (nu - 1 - i) : half;
        const double* k = K + (size_t)(left * (half + 1) + right) * W;
        const double* base = row + (i - left);
        double s = 0.0;
        for (int j = 0; j < left + right + 1; ++j)
            s += __ldg(k + j) * __ldg(base + j);
        orow[i] = s;
    }
}

__global__ void sg_cols_kernel(const double* __restrict__ in, double* __restrict__ out, int nu,
                               int nv, int half, const double* __restrict__ K)
{
    const int W = 2 * half + 1;
    const size_t img = (size_t)blockIdx.z * nu * nv;
    const int iu = blockIdx.x * blockDim.x + threadIdx.x;
    const int iv = blockIdx.y;
    if (iu >= nu)
        return;
    const int left = iv < half ? iv : half;
    const int right = (nv - 1 - iv) < half ? (nv - 1 - iv) : half;
    const double* k = K + (size_t)(left * (half + 1) + right) * W;
    const double* base = in + img + (size_t)(iv - left) * nu + iu;
    double s = 0.0;
    for (int j = 0; j < left + right + 1; ++j)
        s += __ldg(k + j) * __ldg(base + (size_t)j * nu);
    out[img + (size_t)iv * nu + iu] = s;
}

// --------------------------------------------------- angular interpolation
// REF interpolate_angles (postprocess.cpp:147-196): per target image either a
// pass-through (lo == hi, w ignored) or (1-w)*lo + w*hi.

__global__ void interp_kernel(const double* __restrict__ in, double* __restrict__ out,
                              const InterpEntry* __restrict__ tab, size_t npix)
{
    const InterpEntry e = tab[blockIdx.y];
    const double* a = in + (size_t)e.lo * npix;
    const double* b = in + (size_t)e.hi * npix;
    double* o = out + (size_t)blockIdx.y * npix;
    for (size_t p = (size_t)blockIdx.x * blockDim.x + threadIdx.x; p < npix;
         p += (size_t)gridDim.x * blockDim.x) {
        o[p] = e.exact ? __ldg(a + p) : (1.0 - e.w) * __ldg(a + p) + e.w * __ldg(b + p);
    }
}

// ------------------------------------------------------ Catmull-Rom resize
// REF fetch + catmull_rom_pass (postprocess.cpp:201-233).
__device__ __forceinline__ double cr_fetch(const double* line, int n, size_t stride, int i)
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

__device__ __forceinline__ double cr_sample(const double* line, int n_in, int n_out, size_t stride,
                                            int i)
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
    return w0 * cr_fetch(line, n_in, stride, base - 1) + w1 * cr_fetch(line, n_in, stride, base) +
           w2 * cr_fetch(line, n_in, stride, base + 1) + w3 * cr_fetch(line, n_in, stride, base + 2);
}

// rows: in (nv x nu) -> tmp (nv x nu_out)
__global__ void cr_rows_kernel(const double* __restrict__ in, double* __restrict__ tmp, int nu,
                               int nv, int nu_out)
{
    const int iv = blockIdx.y;
    const double* line = in + (size_t)blockIdx.z * nu * nv + (size_t)iv * nu;
    double* o = tmp + (size_t)blockIdx.z * nu_out * nv + (size_t)iv * nu_out;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nu_out; i += gridDim.x * blockDim.x)
        o[i] = cr_sample(line, nu, nu_out, 1, i);
}

// cols: tmp (nv x nu_out) -> out (nv_out x nu_out)
__global__ void cr_cols_kernel(const double* __restrict__ tmp, double* __restrict__ out, int nu_out,
                               int nv, int nv_out)
{
    const int iu = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y;
    if (iu >= nu_out)
        return;
    const double* line = tmp + (size_t)blockIdx.z * nu_out * nv + iu;
    out[(size_t)blockIdx.z * nu_out * nv_out + (size_t)j * nu_out + iu] =
        cr_sample(line, nv, nv_out, (size_t)nu_out, j);
}

// ------------------------------------------------------- block averaging
// REF downsample_average (postprocess.cpp:254-271).
__global__ void downsample_kernel(const double* __restrict__ in, double* __restrict__ out, int nu,
                                  int nv, int nu_out, int nv_out)
{
    const int ou = blockIdx.x * blockDim.x + threadIdx.x;
    const int ov = blockIdx.y;
    if (ou >= nu_out)
        return;
    const double* img = in + (size_t)blockIdx.z * nu * nv;
    const int v0 = ov * nv / nv_out, v1 = (ov + 1) * nv / nv_out;
    const int u0 = ou * nu / nu_out, u1 = (ou + 1) * nu / nu_out;
    double s = 0.0;
    for (int v = v0; v < v1; ++v)
        for (int u = u0; u < u1; ++u)
            s += img[(size_t)v * nu + u];
    out[(size_t)blockIdx.z * nu_out * nv_out + (size_t)ov * nu_out + ou] =
        s / ((v1 - v0) * (u1 - u0));
}

// ---------------------------------------------------------------- launchers
static inline int blocks_for(int n, int b) { return (n + b - 1) / b; }

cudaError_t launch_sg(const double* in, double* tmp, double* out, int nu, int nv, int n_images,
                      int half, const double* K, cudaStream_t s)
{
    dim3 block(128);
    dim3 grid_r(blocks_for(nu, 128), nv, n_images);
    sg_rows_kernel<<<grid_r, block, 0, s>>>(in, tmp, nu, nv, half, K);
    dim3 grid_c(blocks_for(nu, 128), nv, n_images);
    sg_cols_kernel<<<grid_c, block, 0, s>>>(tmp, out, nu, nv, half, K);
    return cudaGetLastError();
}

cudaError_t launch_interp(const double* in, double* out, const InterpEntry* tab, int n_tgt,
                          size_t npix, cudaStream_t s)
{
    int gx = (int)((npix + 255) / 256);
    if (gx > 1024)
        gx = 1024;
    interp_kernel<<<dim3(gx, n_tgt), 256, 0, s>>>(in, out, tab, npix);
    return cudaGetLastError();
}

cudaError_t launch_upsample(const double* in, double* tmp, double* out, int nu, int nv,
                            int n_images, int nu_out, int nv_out, cudaStream_t s)
{
    cr_rows_kernel<<<dim3(blocks_for(nu_out, 128), nv, n_images), 128, 0, s>>>(in, tmp, nu, nv,
                                                                                nu_out);
    cr_cols_kernel<<<dim3(blocks_for(nu_out, 128), nv_out, n_images), 128, 0, s>>>(tmp, out, nu_out,
                                                                                   nv, nv_out);
    return cudaGetLastError();
}

cudaError_t launch_downsample(const double* in, double* out, int nu, int nv, int n_images,
                              int nu_out, int nv_out, cudaStream_t s)
{
    downsample_kernel<<<dim3(blocks_for(nu_out, 128), nv_out, n_images), 128, 0, s>>>(
        in, out, nu, nv, nu_out, nv_out);
    return cudaGetLastError();
}

} // namespace xsd
