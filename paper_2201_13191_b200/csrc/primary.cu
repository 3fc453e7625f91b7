// primary.cu — deterministic primary projector and the tally finalize kernel.
#include <cmath>

#include "physics.cuh"

namespace xsd {

// =========================================================== primary kernel
// REF simulate_primary (transport.cpp:333-377) + trace_rho_lengths
// (trace.cpp:163-187): one thread per pixel, fp64 walk, per-material rho*L in
// shared memory, then the spectrum quadrature with host-tabulated
// attenuation (host glibc loglog, i.e. REF's own values).
template <int FMT>
__global__ void __launch_bounds__(128) primary_kernel(const __grid_constant__ PrimaryParams P)
{
    extern __shared__ __align__(16) unsigned char smem[];
    double* rho = reinterpret_cast<double*>(smem) + threadIdx.x;
    const int stride = blockDim.x;
    const uint64_t pix = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t npix = (uint64_t)P.nu * P.nv;
    if (pix >= npix)
        return;
    const int iv = (int)(pix / (uint64_t)P.nu);
    const int iu = (int)(pix - (uint64_t)iv * P.nu);
    for (int m = 0; m < P.n_mats; ++m)
        rho[m * stride] = 0.0;

    const V3 src = v3(P.src[0], P.src[1], P.src[2]);
    const double du = (iu + 0.5 - 0.5 * P.nu) * P.pitch;
    const double dv = (iv + 0.5 - 0.5 * P.nv) * P.pitch;
    const V3 p = (v3(P.center[0], P.center[1], P.center[2]) + v3(P.uaxis[0], P.uaxis[1], P.uaxis[2]) * du) +
                 v3(0.0, 0.0, 1.0) * dv;
    const V3 delta = p - src;
    const double d2 = dot(delta, delta);
    const V3 d = delta / sqrt(d2);

    const Grid& G = P.G;
    double t0, t1;
    bool bad;
    if (clip_to_grid(G, src, d, t0, t1, bad)) {
        const V3 q = src + d * t0;
        int ix, iy, iz, sx, sy, sz;
        double tnx, tny, tnz, dtx, dty, dtz;
        start_axis(q.x, src.x, d.x, G.ox, G.hx, G.ihx, G.nx, t0, ix, sx, tnx, dtx);
        start_axis(q.y, src.y, d.y, G.oy, G.hy, G.ihy, G.ny, t0, iy, sy, tny, dty);
        start_axis(q.z, src.z, d.z, G.oz, G.hz, G.ihz, G.nz, t0, iz, sz, tnz, dtz);
        double t = t0;
        while (t < t1) {
            double tn = tnx;
            if (tny < tn)
                tn = tny;
            if (tnz < tn)
                tn = tnz;
            if (t1 < tn)
                tn = t1;
            const uint32_t cell = brick_cell(G, ix, iy, iz);
            int m;
            float dens;
            if (FMT == kFmtP4) {
                const int code = load_code_p4(G, cell) & ~G.ubit;
                m = P.pal_mat[code];
                dens = P.pal_dens[code];
            } else if (FMT == kFmtP8) {
                const int code = load_code_p8(G, cell) & ~G.ubit;
                m = P.pal_mat[code];
                dens = P.pal_dens[code];
            } else {
                m = __ldg(G.vox + cell);
                dens = load_density_raw(G, cell);
            }
            rho[m * stride] += (double)dens * (tn - t);
            t = tn;
            if (t >= t1)
                break;
            if (tnx == tn) {
                ix += sx;
                if (ix < 0 || ix >= G.nx)
                    break;
                tnx += dtx;
            }
            if (tny == tn) {
                iy += sy;
                if (iy < 0 || iy >= G.ny)
                    break;
                tny += dty;
            }
            if (tnz == tn) {
                iz += sz;
                if (iz < 0 || iz >= G.nz)
                    break;
                tnz += dtz;
            }
        }
    }
    double value = 0.0;
    for (int b = 0; b < P.n_bins; ++b) {
        double tau = 0.0;
        for (int m = 1; m < P.n_mats; ++m)
            tau += __ldg(P.atten + (size_t)b * P.n_mats + m) * rho[m * stride];
        value += __ldg(P.wresp + b) * __ldg(P.response + b) * exp(-tau) / d2;
    }
    P.image[pix] = value;
}

// ========================================================== finalize kernel
// Limb sums -> fp64 image (+ REF's per-pixel variance, transport.cpp:317-322).
// The accumulator may come in several parts (one per GPU or context of a
// photon-batch split, in local or NVLink peer memory): the kernel sums the
// parts' limbs as it reads them, so the reduce and the finalize are one pass.
constexpr int kMaxSrc = 16;
struct AccSrcs {
    const unsigned long long* p[kMaxSrc];
    int n;
};

__device__ __forceinline__ void load_limbs(const AccSrcs& S, uint64_t off, unsigned long long& l0,
                                           unsigned long long& l1, unsigned long long& l2)
{
    l0 = l1 = l2 = 0ull;
    for (int k = 0; k < S.n; ++k) {
        const ulonglong2 a = *reinterpret_cast<const ulonglong2*>(S.p[k] + off);
        l0 += a.x;
        l1 += a.y;
        l2 += S.p[k][off + 2];
    }
}

__global__ void finalize_image_kernel(const __grid_constant__ AccSrcs S, uint64_t off_image, uint64_t off_var,
                                      uint64_t npix, int log2_img, double n_hist, int track_var,
                                      double* __restrict__ image, double* __restrict__ var)
{
    for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < npix;
         p += (uint64_t)gridDim.x * blockDim.x) {
        unsigned long long l0, l1, l2;
        load_limbs(S, off_image + 4 * p, l0, l1, l2);
        const double v = dequantize(l0, l1, l2, log2_img);
        image[p] = v;
        if (track_var && var) {
            load_limbs(S, off_var + 4 * p, l0, l1, l2);
            const double c2 = dequantize(l0, l1, l2, 2 * log2_img);
            const double x = c2 - v * v / n_hist;
            const double den = 1.0 < n_hist - 1.0 ? n_hist - 1.0 : 1.0;
            var[p] = (0.0 < x ? x : 0.0) * n_hist / den;
        }
    }
}

cudaError_t launch_primary(const PrimaryParams& P, cudaStream_t s)
{
    const int block = 128;
    const uint64_t npix = (uint64_t)P.nu * P.nv;
    const int grid = (int)((npix + block - 1) / block);
    const size_t smem = (size_t)P.n_mats * block * sizeof(double);
    switch (P.G.fmt) {
    case kFmtP4:
        primary_kernel<kFmtP4><<<grid, block, smem, s>>>(P);
        break;
    case kFmtP8:
        primary_kernel<kFmtP8><<<grid, block, smem, s>>>(P);
        break;
    default:
        primary_kernel<kFmtRaw><<<grid, block, smem, s>>>(P);
        break;
    }
    return cudaGetLastError();
}

cudaError_t launch_finalize_image(const unsigned long long* const* srcs, int n_src, uint64_t off_image,
                                  uint64_t off_var, uint64_t npix, int log2_img, double n_hist, int track_var,
                                  double* image, double* var, cudaStream_t s)
{
    if (n_src < 1 || n_src > kMaxSrc)
        return cudaErrorInvalidValue;
    AccSrcs S{};
    S.n = n_src;
    for (int k = 0; k < n_src; ++k)
        S.p[k] = srcs[k];
    const int block = 256;
    int grid = (int)((npix + block - 1) / block);
    if (grid > 148 * 16)
        grid = 148 * 16;
    finalize_image_kernel<<<grid, block, 0, s>>>(S, off_image, off_var, npix, log2_img, n_hist, track_var, image,
                                                 var);
    return cudaGetLastError();
}

} // namespace xsd
