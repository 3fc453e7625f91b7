// transport.cu — Monte Carlo scatter transport, primary projector and the
// tally finalize kernels.
//
// Scatter (REF transport.cpp:114-242 run_history, :246-324 simulate_scatter_stats):
// a persistent kernel; every lane owns one photon history at a time and runs
// the reference's per-history state machine (emission -> exact free-path walk
// -> interaction -> `splitting` next-event scoring rays -> continuation ->
// cap / roulette).  The voxel walks, which are >95 % of the work, run in
// warp-synchronous lockstep: a warp steps all its walking lanes together and
// leaves the walk phase only when enough lanes wait for event processing, at
// which point those lanes advance their state machines and refill from a
// warp-aggregated history pool.  Tallies are fixed-point integers (see
// include/xscat_gpu.h), so the result does not depend on the schedule or on
// how the history range is split across GPUs.
#include <cfloat>
#include <math_constants.h>
#include <cmath>

#include "xs_device.cuh"

namespace xsd {

namespace {

constexpr unsigned kFull = 0xffffffffu;

enum State : int {
    ST_FETCH = 0,
    ST_INIT,
    ST_FREE,
    ST_AFTER_FREE,
    ST_SCORE,
    ST_AFTER_SCORE,
    ST_CONT,
    ST_END,
    ST_WALK,
    ST_DONE
};

enum Kind : int { K_PE = 0, K_COMPTON = 1, K_RAYLEIGH = 2 };

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
    const double st = sin(theta), ct = cos(theta);
    return normalized(dir * ct + (e1 * cos(phi) + e2 * sin(phi)) * st);
}

// ------------------------------------------------------------ physics helpers
__device__ __forceinline__ double momentum_transfer(double e, double theta)
{
    return sin(0.5 * theta) * e / kHc; // cross_sections.cpp:19-22
}

__device__ __forceinline__ double compton_ratio(double e, double theta)
{
    const double alpha = e / kMec2; // cross_sections.cpp:24-28
    return 1.0 / (1.0 + alpha * (1.0 - cos(theta)));
}

__device__ __forceinline__ double kn_core(double e, double theta)
{
    const double ratio = compton_ratio(e, theta);
    const double s = sin(theta);
    return ratio * ratio * (ratio + 1.0 / ratio - s * s);
}

struct Ctx {
    const TransportParams& P;
    DevStatus* st;
};

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

__device__ __forceinline__ double loglog_or_fail(const TransportParams& P, TabDesc d, double e,
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

__device__ double cumulative_mass(const TransportParams& P, const MatDesc& m, double q)
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

__device__ double invert_mass(const TransportParams& P, const MatDesc& m, double target, double q_hi)
{
    double lo = 0.0, hi = q_hi;
    for (int it = 0; it < 64; ++it) {
        const double mid = 0.5 * (lo + hi);
        if (cumulative_mass(P, m, mid) < target)
            lo = mid;
        else
            hi = mid;
    }
    return 0.5 * (lo + hi);
}

// ------------------------------------------------------------- mu tables
// Per-lane table in shared memory, T[k * stride]: for the 4-bit palette the
// linear attenuation of palette entry k (mass_atten[mat_k] * dens_k, the
// same product REF MuField::at forms per voxel); for the other formats the
// mass attenuation of material k (REF MuField, trace.cpp:10-16).
template <int FMT>
__device__ __forceinline__ void fill_mu(const TransportParams& P, double* T, int stride,
                                        double e, DevStatus* st, int bin)
{
    if (FMT == kFmtP4) {
        for (int c = 0; c < P.n_pal; ++c)
            T[c * stride] = 0.0;
        for (int m = 1; m < P.n_mats; ++m) {
            const MatDesc& md = P.mats[m];
            const double ma = md.has_tables ? loglog_or_fail(P, md.mu, e, st, bin) : 0.0;
            for (int c = 0; c < P.n_pal; ++c)
                if (P.pal_mat[c] == m)
                    T[c * stride] = ma * (double)P.pal_dens[c];
        }
    } else {
        T[0] = 0.0;
        for (int m = 1; m < P.n_mats; ++m) {
            const MatDesc& md = P.mats[m];
            T[m * stride] = md.has_tables ? loglog_or_fail(P, md.mu, e, st, bin) : 0.0;
        }
    }
}

template <int FMT>
__device__ __forceinline__ double mu_at(const TransportParams& P, const double* T, int stride,
                                        uint32_t cell)
{
    if (FMT == kFmtP4) {
        return T[load_code_p4(P.G, cell) * stride];
    } else if (FMT == kFmtP8) {
        const int code = load_code_p8(P.G, cell);
        return T[P.pal_mat[code] * stride] * (double)P.pal_dens[code];
    } else {
        const int id = __ldg(P.G.vox + cell);
        return T[id * stride] * (double)load_density_raw(P.G, cell);
    }
}

template <int FMT>
__device__ __forceinline__ int material_at(const TransportParams& P, uint32_t cell)
{
    if (FMT == kFmtP4)
        return P.pal_mat[load_code_p4(P.G, cell)];
    if (FMT == kFmtP8)
        return P.pal_mat[load_code_p8(P.G, cell)];
    return __ldg(P.G.vox + cell);
}

// --------------------------------------------------------------- the walker
// Lane-resident Siddon state (REF trace.cpp:66-103 Walker / start_walk).
struct Walk {
    double rx, ry, rz;        // ray direction (origin = photon position)
    double tnx, tny, tnz;     // next boundary crossing per axis
    double dtx, dty, dtz;     // per-voxel increments (march: dtx = step length)
    double t, texit, depth, target;
    int ix, iy, iz;           // voxel (march: ix = sample j, iy = n samples)
    int sx, sy, sz;
    int march;                // 0 = exact Siddon, 1 = midpoint march (step_voxels > 1)
    int hit;                  // free path: interaction inside the grid
};

// REF clip_to_grid (trace.cpp:29-56); returns false for a miss.
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
        double ta = (l[a] - oo[a]) / dd[a];
        double tb = (h[a] - oo[a]) / dd[a];
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

__device__ __forceinline__ void start_axis(double p, double o, double d, double org, double hs,
                                           double inv_h, int n, double t0, int& idx, int& step,
                                           double& tn, double& dt)
{
    idx = voxel_of(p, org, inv_h, n);
    if (d > 0.0) {
        step = 1;
        dt = hs / d;
        tn = (org + (idx + 1) * hs - o) / d;
    } else if (d < 0.0) {
        step = -1;
        dt = -hs / d;
        tn = (org + idx * hs - o) / d;
    } else {
        step = 0;
        dt = CUDART_INF;
        tn = CUDART_INF;
    }
    while (tn <= t0 && step != 0) {
        idx += step;
        tn += dt;
    }
    // REF leaves an out-of-grid index here only in degenerate tangent cases
    // (it would then read outside the grid); keep the device read in bounds.
    idx = idx < 0 ? 0 : (idx > n - 1 ? n - 1 : idx);
}

// Set up the walk of ray (o, d); returns false if the ray misses the grid.
__device__ __forceinline__ bool walk_begin(const TransportParams& P, Walk& w, V3 o, V3 d,
                                           double target, bool march, DevStatus* st, int bin)
{
    double t0, t1;
    bool bad;
    w.rx = d.x;
    w.ry = d.y;
    w.rz = d.z;
    if (!clip_to_grid(P.G, o, d, t0, t1, bad)) {
        if (bad)
            raise(st, XS_E_INVALID_ARGUMENT, 0, bin, 0.0, 0.0);
        return false;
    }
    w.depth = 0.0;
    w.target = target;
    w.hit = 0;
    w.texit = t1;
    w.t = t0;
    if (march) { // REF trace.cpp:116-134
        w.march = 1;
        const double len = t1 - t0;
        int n = (int)ceil(len / P.march_h);
        w.iy = n < 1 ? 1 : n;
        w.ix = 0;
        w.dtx = P.march_h;
        return true;
    }
    w.march = 0;
    const V3 p = o + d * t0;
    const Grid& G = P.G;
    start_axis(p.x, o.x, d.x, G.ox, G.hx, G.ihx, G.nx, t0, w.ix, w.sx, w.tnx, w.dtx);
    start_axis(p.y, o.y, d.y, G.oy, G.hy, G.ihy, G.ny, t0, w.iy, w.sy, w.tny, w.dty);
    start_axis(p.z, o.z, d.z, G.oz, G.hz, G.ihz, G.nz, t0, w.iz, w.sz, w.tnz, w.dtz);
    return true;
}

// One voxel of the walk.  Returns true while the walk continues.
// Siddon: REF trace.cpp:136-155 (attenuation) / :202-228 (free path).
template <int FMT>
__device__ __forceinline__ bool walk_step(const TransportParams& P, const double* T, int stride,
                                          Walk& w, V3 o)
{
    const Grid& G = P.G;
    if (w.march) {
        const double ta = w.t + w.ix * w.dtx;
        const double tb = w.texit < ta + w.dtx ? w.texit : ta + w.dtx; // std::min
        const double tm = 0.5 * (ta + tb);
        const V3 p = o + v3(w.rx, w.ry, w.rz) * tm;
        const int ix = voxel_of(p.x, G.ox, G.ihx, G.nx);
        const int iy = voxel_of(p.y, G.oy, G.ihy, G.ny);
        const int iz = voxel_of(p.z, G.oz, G.ihz, G.nz);
        w.depth += mu_at<FMT>(P, T, stride, brick_cell(G, ix, iy, iz)) * (tb - ta);
        return ++w.ix < w.iy;
    }
    const double mu = mu_at<FMT>(P, T, stride, brick_cell(G, w.ix, w.iy, w.iz));
    double tn = w.tnx;
    if (w.tny < tn)
        tn = w.tny;
    if (w.tnz < tn)
        tn = w.tnz;
    if (w.texit < tn)
        tn = w.texit;
    const double seg = mu * (tn - w.t);
    if (w.depth + seg >= w.target) { // free path ends inside this voxel
        w.hit = 1;
        w.t = (mu > 0.0) ? w.t + (w.target - w.depth) / mu : tn; // t_hit
        return false;
    }
    w.depth += seg;
    w.t = tn;
    if (w.t >= w.texit)
        return false;
    if (w.tnx == tn) {
        w.ix += w.sx;
        if (w.ix < 0 || w.ix >= G.nx)
            return false;
        w.tnx += w.dtx;
    }
    if (w.tny == tn) {
        w.iy += w.sy;
        if (w.iy < 0 || w.iy >= G.ny)
            return false;
        w.tny += w.dty;
    }
    if (w.tnz == tn) {
        w.iz += w.sz;
        if (w.iz < 0 || w.iz >= G.nz)
            return false;
        w.tnz += w.dtz;
    }
    return true;
}

// ------------------------------------------------------ shared accumulators
struct SAcc {
    unsigned long long* bins;   // n_bins * 8
    unsigned long long* ledger; // 24
    unsigned long long* diag;   // 8
};

__device__ __forceinline__ void sadd(unsigned long long* p, uint64_t v)
{
    if (v)
        atomicAdd(p, (unsigned long long)v);
}

__device__ __forceinline__ bool tally_shared(unsigned long long* slot, double x, int log2_unit)
{
    uint64_t l0, l1, l2;
    if (!quantize(ldexp(x, -log2_unit), l0, l1, l2))
        return false;
    sadd(slot + 0, l0);
    sadd(slot + 1, l1);
    sadd(slot + 2, l2);
    return true;
}

__device__ __forceinline__ void ledger_add(const TransportParams& P, const SAcc& S, int k,
                                           double w, DevStatus* st, int bin)
{
    if (w != 0.0 && !tally_shared(S.ledger + 4 * k, w, P.log2_w))
        raise(st, XS_E_RUNTIME, kErrTallyOverflow, bin, 0.0, w);
}

} // namespace

// =================================================================== kernel
template <int FMT>
__global__ void __launch_bounds__(256, 2) transport_kernel(const __grid_constant__ TransportParams P)
{
    extern __shared__ __align__(16) unsigned char smem[];
    const int n_tab = FMT == kFmtP4 ? P.n_pal : P.n_mats;
    const int stride = blockDim.x;
    double* Tbase = reinterpret_cast<double*>(smem);
    SAcc S;
    S.bins = reinterpret_cast<unsigned long long*>(Tbase + (size_t)n_tab * stride);
    S.ledger = S.bins + 8 * P.n_bins;
    S.diag = S.ledger + 24;
    uint64_t* sstart = reinterpret_cast<uint64_t*>(S.diag + 8);

    for (int i = threadIdx.x; i < 8 * P.n_bins + 32; i += blockDim.x)
        S.bins[i] = 0ull;
    for (int i = threadIdx.x; i <= P.n_bins; i += blockDim.x)
        sstart[i] = P.bin_start[i];
    __syncthreads();

    double* T = Tbase + threadIdx.x;
    DevStatus* st = P.status;
    const int lane = threadIdx.x & 31;
    const unsigned lt_mask = (1u << lane) - 1u;
    const uint64_t gtid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;

    // warp-uniform history queue
    uint64_t wq_next = 0, wq_end = 0;
    bool pool_empty = false;

    // lane state
    int state = ST_FETCH;
    int post = 0; // state to enter when the current walk ends
    Rng rng;
    int bin = 0;
    V3 pos = v3(0, 0, 0), dir = v3(0, 0, 0);
    double energy = 0.0, weight = 0.0, w_min = 0.0, htotal = 0.0, w_split = 0.0, pre = 0.0;
    double T_energy = -1.0;
    int generation = 0, kind = 0, mat = 0, split_left = 0, pixel = 0, n_var = 0;
    uint32_t fp_steps = 0, sc_steps = 0, n_rays = 0, n_inter = 0;
    Walk w;
    w.march = 0;

    const bool march = P.step_voxels > 1;
    const double n_pixels = P.n_pixels;

    for (;;) {
        // ---------------------------------------------------- fetch phase
        unsigned need = __ballot_sync(kFull, state == ST_FETCH);
        while (need) {
            if (wq_next >= wq_end) {
                if (pool_empty) {
                    if (state == ST_FETCH)
                        state = ST_DONE;
                    break;
                }
                unsigned long long base = 0;
                if (lane == 0)
                    base = atomicAdd(P.pool, (unsigned long long)P.grab);
                base = __shfl_sync(kFull, base, 0);
                wq_next = P.h_begin + base;
                wq_end = wq_next + (uint64_t)P.grab;
                if (wq_end > P.h_end)
                    wq_end = P.h_end;
                if (wq_next >= P.h_end) {
                    pool_empty = true;
                    continue;
                }
            }
            const uint64_t avail = wq_end - wq_next;
            const int rank = __popc(need & lt_mask);
            if (state == ST_FETCH && (uint64_t)rank < avail) {
                const uint64_t h = wq_next + rank;
                // bin = last b with start[b] <= h (empty bins are skipped)
                int lo = 0, hi = P.n_bins;
                while (hi - lo > 1) {
                    const int mid = (lo + hi) >> 1;
                    if (sstart[mid] <= h)
                        lo = mid;
                    else
                        hi = mid;
                }
                bin = lo;
                rng_init(rng, (uint32_t)(h - sstart[lo]), (uint32_t)lo);
                state = ST_INIT;
            }
            const uint64_t used = (uint64_t)__popc(need) < avail ? (uint64_t)__popc(need) : avail;
            wq_next += used;
            need = __ballot_sync(kFull, state == ST_FETCH);
        }

        // ---------------------------------------------------- event phase
        while (state != ST_WALK && state != ST_DONE && state != ST_FETCH) {
            switch (state) {
            case ST_INIT: { // REF run_history :120-138, sample_emission :73-87
                const double u1 = rng_uniform(rng, P.k0, P.k1, P.angle);
                const double u2 = rng_uniform(rng, P.k0, P.k1, P.angle);
                const double xu = (u1 - 0.5) * P.nu * P.pitch;
                const double xv = (u2 - 0.5) * P.nv * P.pitch;
                const V3 c = v3(P.center[0], P.center[1], P.center[2]);
                const V3 ua = v3(P.uaxis[0], P.uaxis[1], P.uaxis[2]);
                const V3 target = (c + ua * xu) + v3(0.0, 0.0, 1.0) * xv;
                const V3 src = v3(P.src[0], P.src[1], P.src[2]);
                const V3 delta = target - src;
                const double d2 = dot(delta, delta);
                dir = delta / sqrt(d2);
                const double cos_psi = -dot(dir, v3(P.normal[0], P.normal[1], P.normal[2]));
                const double em_weight = P.det_area * cos_psi / d2;
                const double w0 = __ldg(P.bin_weight + bin) * em_weight / (double)__ldg(P.bin_count + bin);
                w_min = P.wmin_rel * w0;
                pos = src;
                energy = __ldg(P.bin_energy + bin);
                weight = w0;
                generation = 0;
                htotal = 0.0;
                n_var = 0;
                ledger_add(P, S, 0, w0, st, bin);
                if (T_energy != energy) {
                    fill_mu<FMT>(P, T, stride, energy, st, bin);
                    T_energy = energy;
                }
                state = ST_FREE;
                break;
            }
            case ST_FREE: { // REF trace.cpp:189-230 sample_free_path
                const double u = rng_uniform(rng, P.k0, P.k1, P.angle);
                if (T_energy != energy) {
                    fill_mu<FMT>(P, T, stride, energy, st, bin);
                    T_energy = energy;
                }
                if (walk_begin(P, w, pos, dir, -log(u), false, st, bin)) {
                    post = ST_AFTER_FREE;
                    state = ST_WALK;
                } else {
                    w.hit = 0;
                    state = ST_AFTER_FREE;
                }
                break;
            }
            case ST_AFTER_FREE: { // REF run_history :141-160
                if (!w.hit) {
                    ledger_add(P, S, 1, weight, st, bin);
                    state = ST_END;
                    break;
                }
                const uint32_t cell = brick_cell(P.G, w.ix, w.iy, w.iz);
                pos = pos + v3(w.rx, w.ry, w.rz) * w.t;
                mat = material_at<FMT>(P, cell);
                ++n_inter;
                const MatDesc& md = P.mats[mat];
                // select_interaction (cross_sections.cpp:81-96)
                const double pe = loglog_or_fail(P, md.pe, energy, st, bin);
                const double incoh = loglog_or_fail(P, md.incoh, energy, st, bin);
                const double coh = loglog_or_fail(P, md.coh, energy, st, bin);
                const double total = pe + incoh + coh;
                if (!(total > 0.0))
                    raise(st, XS_E_RUNTIME, kErrSigmaAll, bin, energy, (double)mat);
                const double u = rng_uniform(rng, P.k0, P.k1, P.angle) * total;
                kind = u < pe ? K_PE : (u < pe + incoh ? K_COMPTON : K_RAYLEIGH);
                if (kind == K_PE) {
                    ledger_add(P, S, 2, weight, st, bin);
                    state = ST_END;
                    break;
                }
                w_split = weight / P.splitting;
                split_left = P.splitting;
                state = ST_SCORE;
                break;
            }
            case ST_SCORE: { // REF run_history :162-183
                int iu = (int)(rng_uniform(rng, P.k0, P.k1, P.angle) * P.nu);
                int iv = (int)(rng_uniform(rng, P.k0, P.k1, P.angle) * P.nv);
                iu = iu < P.nu - 1 ? iu : P.nu - 1;
                iv = iv < P.nv - 1 ? iv : P.nv - 1;
                const double du = (iu + 0.5 - 0.5 * P.nu) * P.pitch;
                const double dv = (iv + 0.5 - 0.5 * P.nv) * P.pitch;
                const V3 c = v3(P.center[0], P.center[1], P.center[2]);
                const V3 ua = v3(P.uaxis[0], P.uaxis[1], P.uaxis[2]);
                const V3 pix = (c + ua * du) + v3(0.0, 0.0, 1.0) * dv;
                const V3 delta = pix - pos;
                const double d2 = dot(delta, delta);
                const V3 to_det = delta / sqrt(d2);
                double cos_t = dot(dir, to_det);
                cos_t = cos_t < -1.0 ? -1.0 : (1.0 < cos_t ? 1.0 : cos_t);
                const double theta = acos(cos_t);
                const MatDesc& md = P.mats[mat];
                double p_dir, e_out;
                const double r0 = kR0;
                if (kind == K_COMPTON) { // cross_sections.cpp:56-66
                    const double sigma = loglog_or_fail(P, md.incoh, energy, st, bin) * kBarn;
                    if (!(sigma > 0.0))
                        raise(st, XS_E_RUNTIME, kErrSigmaIncoh, bin, energy, 0.0);
                    p_dir = kPi * r0 * r0 / sigma * kn_core(energy, theta) *
                            form_S(P, md, momentum_transfer(energy, theta));
                    e_out = energy * compton_ratio(energy, theta);
                } else { // cross_sections.cpp:68-79
                    const double sigma = loglog_or_fail(P, md.coh, energy, st, bin) * kBarn;
                    if (!(sigma > 0.0))
                        raise(st, XS_E_RUNTIME, kErrSigmaCoh, bin, energy, 0.0);
                    const double c2 = cos(theta);
                    const double f = form_F(P, md, momentum_transfer(energy, theta));
                    p_dir = kPi * r0 * r0 / sigma * (1.0 + c2 * c2) * f * f;
                    e_out = energy;
                }
                double dep = 0.0;
                if (!tab_linear(mtab(P, P.resp_deposit), e_out, dep))
                    raise(st, XS_E_OUT_OF_RANGE, kErrTableRange, bin, e_out, 1.0);
                const double rf = dep / e_out;
                // REF point_detector_score :66-71 without the exp(-tau) factor
                pre = rf * p_dir * w_split * n_pixels / (2.0 * kPi * d2);
                pixel = iv * P.nu + iu;
                if (T_energy != e_out) { // REF trace_attenuation builds MuField(e_out)
                    fill_mu<FMT>(P, T, stride, e_out, st, bin);
                    T_energy = e_out;
                }
                ++n_rays;
                if (walk_begin(P, w, pos, to_det, CUDART_INF, march, st, bin)) {
                    post = ST_AFTER_SCORE;
                    state = ST_WALK;
                } else {
                    w.depth = 0.0;
                    state = ST_AFTER_SCORE;
                }
                break;
            }
            case ST_AFTER_SCORE: { // REF run_history :178-193
                const double x = pre * exp(-w.depth);
                if (!isfinite(x))
                    raise(st, XS_E_RUNTIME, kErrNonFinite, bin, energy, x);
                else if (!tally_global(P.accum + P.off_image + 4ull * (uint64_t)pixel, x, P.log2_img))
                    raise(st, XS_E_RUNTIME, kErrTallyOverflow, bin, energy, x);
                htotal += x;
                if (P.track_var && n_var < P.var_cap) {
                    P.var_pix[gtid * P.var_cap + n_var] = (uint32_t)pixel;
                    P.var_val[gtid * P.var_cap + n_var] = x;
                    ++n_var;
                }
                state = --split_left > 0 ? ST_SCORE : ST_CONT;
                break;
            }
            case ST_CONT: { // REF run_history :195-223
                const MatDesc& md = P.mats[mat];
                if (kind == K_COMPTON) { // samplers.cpp:32-52
                    const double alpha = energy / kMec2;
                    const double q_max = momentum_transfer(energy, kPi);
                    const double s_max = form_S(P, md, q_max);
                    if (!(s_max > 0.0)) {
                        raise(st, XS_E_RUNTIME, kErrComptonS, bin, energy, 0.0);
                        state = ST_END;
                        break;
                    }
                    double theta = 0.0, ap = 0.0, phi = 0.0;
                    for (;;) {
                        // kahn_sample_cos_theta (samplers.cpp:12-30)
                        const double t = 1.0 + 2.0 * alpha;
                        double cos_th;
                        for (;;) {
                            const double r1 = rng_uniform(rng, P.k0, P.k1, P.angle);
                            const double r2 = rng_uniform(rng, P.k0, P.k1, P.angle);
                            const double r3 = rng_uniform(rng, P.k0, P.k1, P.angle);
                            if (r1 <= t / (t + 8.0)) {
                                const double x = 1.0 + 2.0 * alpha * r2;
                                if (r3 <= 4.0 * (1.0 / x - 1.0 / (x * x))) {
                                    cos_th = 1.0 - (x - 1.0) / alpha;
                                    break;
                                }
                            } else {
                                const double x = t / (1.0 + 2.0 * alpha * r2);
                                const double ct = 1.0 - (x - 1.0) / alpha;
                                if (r3 <= 0.5 * (ct * ct + 1.0 / x)) {
                                    cos_th = ct;
                                    break;
                                }
                            }
                        }
                        const double cc = cos_th < -1.0 ? -1.0 : (1.0 < cos_th ? 1.0 : cos_th);
                        theta = acos(cc);
                        const double s = form_S(P, md, momentum_transfer(energy, theta));
                        if (rng_uniform(rng, P.k0, P.k1, P.angle) * s_max <= s) {
                            ap = alpha / (1.0 + alpha * (1.0 - cos(theta)));
                            phi = 2.0 * kPi * rng_uniform(rng, P.k0, P.k1, P.angle);
                            break;
                        }
                    }
                    dir = rotate_direction(dir, theta, phi);
                    energy = ap * kMec2;
                } else { // samplers.cpp:106-125
                    const double q_max = momentum_transfer(energy, kPi);
                    const double total = cumulative_mass(P, md, q_max);
                    if (!(total > 0.0)) {
                        raise(st, XS_E_RUNTIME, kErrRayleighF, bin, energy, 0.0);
                        state = ST_END;
                        break;
                    }
                    const double scale = kHc / energy;
                    double theta = 0.0, phi = 0.0;
                    for (;;) {
                        const double q =
                            invert_mass(P, md, rng_uniform(rng, P.k0, P.k1, P.angle) * total, q_max);
                        const double sh = 1.0 < q * scale ? 1.0 : q * scale;
                        const double cos_th = 1.0 - 2.0 * sh * sh;
                        if (rng_uniform(rng, P.k0, P.k1, P.angle) * 2.0 <= 1.0 + cos_th * cos_th) {
                            const double cc = cos_th < -1.0 ? -1.0 : (1.0 < cos_th ? 1.0 : cos_th);
                            theta = acos(cc);
                            phi = 2.0 * kPi * rng_uniform(rng, P.k0, P.k1, P.angle);
                            break;
                        }
                    }
                    dir = rotate_direction(dir, theta, phi);
                }
                ++generation;
                if (generation >= P.max_inter) {
                    ledger_add(P, S, 3, weight, st, bin);
                    state = ST_END;
                    break;
                }
                if (w_min > 0.0 && weight < w_min) {
                    if (rng_uniform(rng, P.k0, P.k1, P.angle) < P.survival) {
                        const double boosted = weight / P.survival;
                        ledger_add(P, S, 5, boosted - weight, st, bin);
                        weight = boosted;
                    } else {
                        ledger_add(P, S, 4, weight, st, bin);
                        state = ST_END;
                        break;
                    }
                }
                state = ST_FREE;
                break;
            }
            case ST_END: { // REF run_history :225-241
                unsigned long long* bs = S.bins + 8 * bin;
                if (htotal != 0.0) {
                    if (!tally_shared(bs, htotal, P.log2_img) ||
                        !tally_shared(bs + 3, htotal * htotal, 2 * P.log2_img))
                        raise(st, XS_E_RUNTIME, kErrTallyOverflow, bin, energy, htotal);
                }
                if (P.track_var) {
                    const uint32_t* vp = P.var_pix + gtid * P.var_cap;
                    const double* vv = P.var_val + gtid * P.var_cap;
                    for (int a = 0; a < n_var; ++a) {
                        const uint32_t pa = vp[a];
                        bool dup = false;
                        for (int b2 = 0; b2 < a; ++b2)
                            if (vp[b2] == pa) {
                                dup = true;
                                break;
                            }
                        if (dup)
                            continue;
                        double c = vv[a];
                        for (int b2 = a + 1; b2 < n_var; ++b2)
                            if (vp[b2] == pa)
                                c += vv[b2];
                        if (!tally_global(P.accum + P.off_var + 4ull * pa, c * c, 2 * P.log2_img))
                            raise(st, XS_E_RUNTIME, kErrTallyOverflow, bin, energy, c);
                    }
                }
                sadd(S.diag + 0, fp_steps);
                sadd(S.diag + 1, sc_steps);
                sadd(S.diag + 2, 1);
                sadd(S.diag + 3, n_rays);
                sadd(S.diag + 4, n_inter);
                fp_steps = sc_steps = n_rays = n_inter = 0;
                // abort the launch on the first device error
                state = *(volatile int32_t*)&st->code != 0 ? ST_DONE : ST_FETCH;
                break;
            }
            default:
                state = ST_DONE;
                break;
            }
        }

        // ----------------------------------------------------- walk phase
        unsigned walking = __ballot_sync(kFull, state == ST_WALK);
        if (!walking) {
            if (__ballot_sync(kFull, state != ST_DONE) == 0)
                break;
            continue;
        }
        for (;;) {
            if (state == ST_WALK) {
                const bool go = walk_step<FMT>(P, T, stride, w, pos);
                if (post == ST_AFTER_FREE)
                    ++fp_steps;
                else
                    ++sc_steps;
                if (!go)
                    state = post;
            }
            walking = __ballot_sync(kFull, state == ST_WALK);
            if (!walking)
                break;
            const unsigned waiting = __ballot_sync(kFull, state != ST_WALK && state != ST_DONE);
            if (__popc(waiting) >= P.walk_thresh)
                break;
        }
    }

    // flush the block's statistics
    __syncthreads();
    for (int i = threadIdx.x; i < 8 * P.n_bins; i += blockDim.x)
        red_add(P.accum + P.off_bins + i, S.bins[i]);
    for (int i = threadIdx.x; i < 24; i += blockDim.x)
        red_add(P.accum + P.off_ledger + i, S.ledger[i]);
    for (int i = threadIdx.x; i < 8; i += blockDim.x)
        red_add(P.accum + P.off_diag + i, S.diag[i]);
}

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
                const int code = load_code_p4(G, cell);
                m = P.pal_mat[code];
                dens = P.pal_dens[code];
            } else if (FMT == kFmtP8) {
                const int code = load_code_p8(G, cell);
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
__global__ void finalize_image_kernel(const unsigned long long* __restrict__ acc, uint64_t off_image,
                                      uint64_t off_var, uint64_t npix, int log2_img, double n_hist,
                                      int track_var, double* __restrict__ image,
                                      double* __restrict__ var)
{
    for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < npix;
         p += (uint64_t)gridDim.x * blockDim.x) {
        const ulonglong2 a = *reinterpret_cast<const ulonglong2*>(acc + off_image + 4 * p);
        const double v = dequantize(a.x, a.y, acc[off_image + 4 * p + 2], log2_img);
        image[p] = v;
        if (track_var && var) {
            const double c2 = dequantize(acc[off_var + 4 * p], acc[off_var + 4 * p + 1],
                                         acc[off_var + 4 * p + 2], 2 * log2_img);
            const double x = c2 - v * v / n_hist;
            const double den = 1.0 < n_hist - 1.0 ? n_hist - 1.0 : 1.0;
            var[p] = (0.0 < x ? x : 0.0) * n_hist / den;
        }
    }
}

// ----------------------------------------------------------------- launchers
cudaError_t launch_transport(const TransportParams& P, int grid, int block, size_t smem,
                             cudaStream_t s)
{
    switch (P.G.fmt) {
    case kFmtP4:
        transport_kernel<kFmtP4><<<grid, block, smem, s>>>(P);
        break;
    case kFmtP8:
        transport_kernel<kFmtP8><<<grid, block, smem, s>>>(P);
        break;
    default:
        transport_kernel<kFmtRaw><<<grid, block, smem, s>>>(P);
        break;
    }
    return cudaGetLastError();
}

cudaError_t transport_set_smem(size_t smem)
{
    cudaError_t e;
    if ((e = cudaFuncSetAttribute(transport_kernel<kFmtP4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem)) != cudaSuccess)
        return e;
    if ((e = cudaFuncSetAttribute(transport_kernel<kFmtP8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem)) != cudaSuccess)
        return e;
    return cudaFuncSetAttribute(transport_kernel<kFmtRaw>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem);
}

cudaError_t transport_occupancy(int fmt, int block, size_t smem, int* blocks_per_sm)
{
    switch (fmt) {
    case kFmtP4:
        return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, transport_kernel<kFmtP4>,
                                                             block, smem);
    case kFmtP8:
        return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, transport_kernel<kFmtP8>,
                                                             block, smem);
    default:
        return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, transport_kernel<kFmtRaw>,
                                                             block, smem);
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

cudaError_t launch_finalize_image(const unsigned long long* acc, uint64_t off_image, uint64_t off_var,
                                  uint64_t npix, int log2_img, double n_hist, int track_var,
                                  double* image, double* var, cudaStream_t s)
{
    const int block = 256;
    int grid = (int)((npix + block - 1) / block);
    if (grid > 148 * 16)
        grid = 148 * 16;
    finalize_image_kernel<<<grid, block, 0, s>>>(acc, off_image, off_var, npix, log2_img, n_hist,
                                                 track_var, image, var);
    return cudaGetLastError();
}

} // namespace xsd
