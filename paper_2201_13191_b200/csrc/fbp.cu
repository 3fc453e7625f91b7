// fbp.cu — FDK reconstruction on the device (REF fbp_reconstruct,
// recon.cpp:58-157).
//
// Same arithmetic and summation order as REF, so the float volume is
// bit-identical:
//   * filter: cosine pre-weighting, then the direct row convolution with the
//     (Hann-windowed) ramp kernel, each output summed over j = 0..nu-1 in
//     order, times du.  Register tiling: a thread owns T outputs and walks j
//     in steps of T with the 2T-1 kernel taps of the step in registers, so
//     one T x T tile costs 3T - 1 shared-memory loads for T^2 fp64 MACs; the
//     kernel taps are stored with a one-word skew per 8 so the loads are free
//     of bank conflicts.
//   * backprojection: one thread per voxel, views in REF's order, each view's
//     contribution formed in fp64 and added to a float accumulator exactly
//     like REF's `vol.at(...) += static_cast<float>(...)`.
// cos / sin of the view angles and the ramp kernel come from the host (glibc,
// REF's own formulas).
#include <cstdint>

#include "xs_types.h"

namespace xsd {

namespace {

constexpr int kT = 8;         // outputs per thread in the filter
constexpr int kFiltThr = 256; // threads per filter block

// grid: (view, row group); dynamic smem: padded kernel (2nu-1 + 2(kT-1)) + row (nu + kT)
__global__ void __launch_bounds__(kFiltThr) fbp_filter_kernel(const double* __restrict__ in,
                                                               double* __restrict__ out,
                                                               const double* __restrict__ kern, int nu, int nv,
                                                               int rows_per_block, double R, double du, double dv)
{
    extern __shared__ double sm[];
    // logical K[k] = kernel[k - (kT - 1)] (zero outside), stored at k + k / 8:
    // a thread reads taps 8 apart from its neighbour, and the one-word skew
    // per 8 spreads a half-warp's 64-bit loads over all banks (stride 9)
    double* K = sm;
    const int nk = 2 * nu - 1 + 2 * (kT - 1);
    double* row = sm + nk + nk / 8 + 1; // nu entries + kT zero tail
    for (int m = threadIdx.x; m < nk; m += blockDim.x) {
        const int src = m - (kT - 1);
        K[m + (m >> 3)] = (src >= 0 && src < 2 * nu - 1) ? kern[src] : 0.0;
    }
    const int view = blockIdx.x;
    const double* img = in + (size_t)view * nu * nv;
    double* q = out + (size_t)view * nu * nv;
    const int r0 = blockIdx.y * rows_per_block, r1 = min(nv, r0 + rows_per_block);
    for (int iv = r0; iv < r1; ++iv) {
        __syncthreads(); // previous row's readers done (and K ready)
        const double vv = (iv + 0.5 - 0.5 * nv) * dv;
        for (int iu = threadIdx.x; iu < nu + kT; iu += blockDim.x) {
            double w = 0.0;
            if (iu < nu) { // REF recon.cpp:93-99
                const double uu = (iu + 0.5 - 0.5 * nu) * du;
                w = img[(size_t)iv * nu + iu] * R / sqrt(R * R + uu * uu + vv * vv);
            }
            row[iu] = w;
        }
        __syncthreads();
        for (int i0 = threadIdx.x * kT; i0 < nu; i0 += blockDim.x * kT) {
            double s[kT];
#pragma unroll
            for (int t = 0; t < kT; ++t)
                s[t] = 0.0;
            // output i = i0 + t, tap j: kernel[i - j + nu - 1] = K[i - j + nu - 1 + kT - 1];
            // tile (i0 + t, j0 + u) uses kk[t - u + kT - 1] = K[kb + m], kb = i0 - j0 + nu - 1
            const int r = (nu - 1) & 7; // kb mod 8 (i0, j0 are multiples of kT = 8)
            for (int j0 = 0; j0 < nu; j0 += kT) {
                const int kb = i0 - j0 + nu - 1;
                const double* kp = K + kb + (kb >> 3);
                double kk[2 * kT - 1]; // kk[m] = K[kb + m] at kb + m + (kb + m) / 8
#pragma unroll
                for (int m = 0; m < 2 * kT - 1; ++m)
                    kk[m] = kp[m + ((r + m) >> 3)];
                if (j0 + kT <= nu) {
#pragma unroll
                    for (int u = 0; u < kT; ++u) {
                        const double r = row[j0 + u];
#pragma unroll
                        for (int t = 0; t < kT; ++t)
                            s[t] += r * kk[t - u + kT - 1];
                    }
                } else { // last partial step: exactly REF's nu terms
#pragma unroll
                    for (int u = 0; u < kT; ++u) {
                        if (j0 + u < nu) {
                            const double r = row[j0 + u];
#pragma unroll
                            for (int t = 0; t < kT; ++t)
                                s[t] += r * kk[t - u + kT - 1];
                        }
                    }
                }
            }
#pragma unroll
            for (int t = 0; t < kT; ++t)
                if (i0 + t < nu)
                    q[(size_t)iv * nu + i0 + t] = s[t] * du;
        }
    }
}

struct BpView {
    double cb, sb, dbeta;
};

// grid: (x blocks, y, z); dynamic smem: n_views BpView
__global__ void fbp_backproject_kernel(const double* __restrict__ q, const BpView* __restrict__ views, int n_views,
                                       int nu, int nv, int nx, int ny, double vx, double vy, double vz, double x0,
                                       double y0, double z0, double R, double du, double dv,
                                       float* __restrict__ vol)
{
    extern __shared__ BpView sv[];
    for (int i = threadIdx.x; i < n_views; i += blockDim.x)
        sv[i] = views[i];
    __syncthreads();
    const int ix = blockIdx.x * blockDim.x + threadIdx.x;
    if (ix >= nx)
        return;
    const int iy = blockIdx.y, iz = blockIdx.z;
    const double z = z0 + (iz + 0.5) * vz;
    const double y = y0 + (iy + 0.5) * vy;
    const double x = x0 + (ix + 0.5) * vx;
    float acc = 0.0f;
    for (int view = 0; view < n_views; ++view) { // REF recon.cpp:121-150
        const double cb = sv[view].cb, sb = sv[view].sb;
        const double* qv = q + (size_t)view * nu * nv;
        const double s_comp = x * cb + y * sb;
        const double t_comp = -x * sb + y * cb;
        const double L = R - s_comp;
        if (L <= 1e-9)
            continue;
        const double pu = (R * t_comp / L) / du + 0.5 * nu - 0.5;
        const double pv = (R * z / L) / dv + 0.5 * nv - 0.5;
        if (pu < 0.0 || pu > nu - 1 || pv < 0.0 || pv > nv - 1)
            continue;
        const int u0 = min((int)pu, nu - 2);
        const int v0 = min((int)pv, nv - 2);
        const double fu = pu - u0, fv = pv - v0;
        const double val = (1 - fu) * (1 - fv) * qv[(size_t)v0 * nu + u0] +
                           fu * (1 - fv) * qv[(size_t)v0 * nu + u0 + 1] +
                           (1 - fu) * fv * qv[(size_t)(v0 + 1) * nu + u0] +
                           fu * fv * qv[(size_t)(v0 + 1) * nu + u0 + 1];
        acc += static_cast<float>(sv[view].dbeta * R * R / (L * L) * val);
    }
    vol[(size_t)ix + (size_t)nx * ((size_t)iy + (size_t)ny * iz)] = acc * 100.0f; // 1/cm -> 1/m
}

} // namespace

size_t fbp_filter_smem(int nu)
{
    const int nk = 2 * nu - 1 + 2 * (kT - 1);
    return (size_t)(nk + nk / 8 + 1 + nu + kT) * sizeof(double);
}

cudaError_t launch_fbp_filter(const double* in, double* out, const double* kern, int nu, int nv, int n_views,
                              double R, double du, double dv, cudaStream_t s)
{
    const size_t smem = fbp_filter_smem(nu);
    cudaError_t e = cudaFuncSetAttribute(fbp_filter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess)
        return e;
    const int rows_per_block = 8;
    const dim3 grid(n_views, (nv + rows_per_block - 1) / rows_per_block);
    fbp_filter_kernel<<<grid, kFiltThr, smem, s>>>(in, out, kern, nu, nv, rows_per_block, R, du, dv);
    return cudaGetLastError();
}

cudaError_t launch_fbp_backproject(const double* q, const void* views, int n_views, int nu, int nv,
                                   const int dims[3], const double voxel[3], double R, double du, double dv,
                                   float* vol, cudaStream_t s)
{
    const size_t smem = (size_t)n_views * sizeof(BpView);
    cudaError_t e =
        cudaFuncSetAttribute(fbp_backproject_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess)
        return e;
    const double x0 = -0.5 * dims[0] * voxel[0]; // REF recon.cpp:114-116
    const double y0 = -0.5 * dims[1] * voxel[1];
    const double z0 = -0.5 * dims[2] * voxel[2];
    const dim3 grid((dims[0] + 127) / 128, dims[1], dims[2]);
    fbp_backproject_kernel<<<grid, 128, smem, s>>>(q, static_cast<const BpView*>(views), n_views, nu, nv, dims[0],
                                                    dims[1], voxel[0], voxel[1], voxel[2], x0, y0, z0, R, du, dv,
                                                    vol);
    return cudaGetLastError();
}

} // namespace xsd
