// transport.cu — Monte Carlo scatter transport (REF transport.cpp:114-324).
//
// Design (B200): a persistent kernel whose warps are independent "ray
// engines".  Each warp owns, in shared memory,
//   * H history slots: the photon state of a live history (position,
//     direction, energy, weight, its Philox stream) plus the record of its
//     last interaction, and
//   * a FIFO of ray tasks (8 bytes each): "free path of history s" or
//     "next-event scoring ray of history s towards pixel p".
// A history's event logic (REF run_history) runs when its free-path ray
// completes: it samples the interaction, draws the `splitting` scoring pixels
// (same Philox order as REF), pushes one scoring task per pixel, samples the
// continuation and pushes its next free path.  Scoring rays do not change the
// photon, so they are fire-and-forget tasks that any lane of the warp traces.
// All 32 lanes therefore pull independent rays from one queue and walk them in
// lockstep, which keeps the SIMT lanes busy (a one-history-per-lane design
// idles most of them; see profiles/).  FIFO order guarantees that the
// scoring rays of an interaction start (and copy its record) before the
// history's next free path can complete and overwrite it.
//
// Tallies are fixed-point integers (include/xscat_gpu.h): per-pixel limbs in
// global memory, per-history totals in the slot, per-bin and ledger sums in
// shared memory, so results are independent of the schedule and of how the
// history range is split across GPUs.
#include <cmath>

#include "physics.cuh"

namespace xsd {

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kWarps = 4; // warps per block
constexpr int kBlock = 32 * kWarps;
#ifndef XSD_MIN_BLOCKS
#define XSD_MIN_BLOCKS 4
#endif

enum : int { T_NONE = -1, T_FREE = 0, T_SCORE = 1 };
enum : int { K_PE = 0, K_COMPTON = 1, K_RAYLEIGH = 2 };

// ------------------------------------------------------------ smem layout
struct __align__(8) Slot {
    double px, py, pz, dx, dy, dz; // photon position (= last interaction point) / direction
    double E, W, wmin, target;     // energy, weight, roulette floor, -ln u of the pending free path
    double ix, iy, iz;             // incoming direction at it
    double e_in, w_split;          // energy at it, weight per pseudo-particle
    double pref;                   // pi r0^2 / sigma(E) of its kind (REF cross_sections.cpp:56-79)
    unsigned long long T[3];       // history total, fixed-point limbs (unit U_img)
    uint32_t r_photon, r_bin, r_block, r_pos, r_b0, r_b1, r_b2, r_b3; // Philox stream
    int32_t bin, gen, kind, mat;
    int32_t pending;               // queued/in-flight scoring rays + 1 while alive
    int32_t n_var;                 // variance scratch entries
};

// Two per-warp FIFOs: scoring rays (H * splitting entries) and free paths
// (kFreeQ >= H entries, right after the scoring FIFO).  Batches are filled
// scoring-first, so a batch is mostly one kind of ray (similar lengths, fewer
// idle lanes in the lockstep walk).  Safety of the record reuse: a free path
// is only popped once every scoring ray queued before it has been popped,
// and set-up (which reads the interaction record) precedes any completion.
constexpr int kFreeQ = 64;
struct WarpHdr {
    uint32_t tail;  // scoring FIFO
    uint32_t ftail; // free-path FIFO
    unsigned long long free_mask;
};

// One out-of-line Philox draw on a history's stream kept in its slot (REF
// rng.hpp:29-60).  A single copy of the 10-round refill instead of one per
// call site keeps the event code small (instruction-cache bound kernel).
__device__ __noinline__ double slot_uniform(Slot* s, uint32_t k0, uint32_t k1, uint32_t angle)
{
    if (s->r_pos == 4) {
        uint32_t c0 = s->r_block, c1 = s->r_photon, c2 = s->r_bin, c3 = angle;
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
        s->r_b0 = c0;
        s->r_b1 = c1;
        s->r_b2 = c2;
        s->r_b3 = c3;
        s->r_pos = 0;
        ++s->r_block;
    }
    uint64_t hi, lo;
    if (s->r_pos == 0) {
        hi = s->r_b0;
        lo = s->r_b1;
    } else {
        hi = s->r_b2;
        lo = s->r_b3;
    }
    s->r_pos += 2;
    const uint64_t bits = ((hi << 32) | lo) >> 11;
    return ((double)bits + 0.5) * 0x1p-53;
}

__device__ __forceinline__ Rng load_rng(const Slot& s)
{
    Rng r;
    r.photon = s.r_photon;
    r.bin = s.r_bin;
    r.block = s.r_block;
    r.pos = s.r_pos;
    r.b0 = s.r_b0;
    r.b1 = s.r_b1;
    r.b2 = s.r_b2;
    r.b3 = s.r_b3;
    return r;
}

__device__ __forceinline__ void store_rng(Slot& s, const Rng& r)
{
    s.r_photon = r.photon;
    s.r_bin = r.bin;
    s.r_block = r.block;
    s.r_pos = r.pos;
    s.r_b0 = r.b0;
    s.r_b1 = r.b1;
    s.r_b2 = r.b2;
    s.r_b3 = r.b3;
}

// ----------------------------------------------------------------- mu table
// Linear attenuation lookup for the current ray's energy.  REG: <= 4 palette
// entries held in registers (4-bit palette); otherwise a per-lane table in
// shared memory: palette entries (P4) or mass attenuation per material
// (P8 / raw, multiplied by the voxel density at lookup).  Values are the
// products REF MuField forms (trace.cpp:10-20).
// Log-log evaluation of several tables at one energy.  When every material's
// mu table has the same energy knots (true for the reference's bundled data,
// checked at upload) the knot search and log(e) are shared; the arithmetic
// is that of tab_loglog (REF table.hpp:57-69), so values are identical.
struct SharedLog {
    int i;
    bool exact, ok;
    double le;
    __device__ __forceinline__ void init(const TransportParams& P, double e, DevStatus* st, int bin)
    {
        ok = false;
        if (!P.shared_mu_grid)
            return;
        const Tab t = mtab(P, P.mats[P.grid_mat].mu);
        if (!tab_locate(t, e, i, exact)) {
            raise(st, XS_E_OUT_OF_RANGE, kErrTableRange, bin, e, 0.0);
            return;
        }
        le = exact ? 0.0 : nl_log(e);
        ok = true;
    }
    __device__ __forceinline__ double eval(const TransportParams& P, TabDesc d, double e, DevStatus* st,
                                           int bin) const
    {
        if (!ok)
            return loglog_or_fail(P, d, e, st, bin);
        const Tab t = mtab(P, d);
        if (exact)
            return __ldg(t.y + i);
        const double y0 = __ldg(t.y + i), y1 = __ldg(t.y + i + 1);
        if (y0 <= 0.0 || y1 <= 0.0) {
            const double x0 = __ldg(t.x + i), x1 = __ldg(t.x + i + 1);
            const double u = (e - x0) / (x1 - x0);
            return y0 + u * (y1 - y0);
        }
        const double lx0 = __ldg(t.lx + i), lx1 = __ldg(t.lx + i + 1);
        const double u = (le - lx0) / (lx1 - lx0);
        return nl_exp(__ldg(t.ly + i) + u * (__ldg(t.ly + i + 1) - __ldg(t.ly + i)));
    }
};

template <int FMT, bool REG>
struct MuTab {
    double t0, t1, t2, t3;
    double* T;
    double energy;

    __device__ __noinline__ void fill(const TransportParams& P, double e, DevStatus* st, int bin)
    {
        energy = e;
        if (FMT == kFmtP4) {
            double v0 = 0.0, v1 = 0.0, v2 = 0.0, v3_ = 0.0;
            if (!REG)
                for (int c = 0; c < P.n_pal; ++c)
                    T[c * kBlock] = 0.0;
            SharedLog sl;
            sl.init(P, e, st, bin);
            for (int m = 1; m < P.n_mats; ++m) {
                const MatDesc& md = P.mats[m];
                const double ma = md.has_tables ? sl.eval(P, md.mu, e, st, bin) : 0.0;
                for (int c = 0; c < P.n_pal; ++c)
                    if (P.pal_mat[c] == m) {
                        const double mu = ma * (double)P.pal_dens[c];
                        if (REG) {
                            if (c == 0)
                                v0 = mu;
                            else if (c == 1)
                                v1 = mu;
                            else if (c == 2)
                                v2 = mu;
                            else
                                v3_ = mu;
                        } else {
                            T[c * kBlock] = mu;
                        }
                    }
            }
            t0 = v0;
            t1 = v1;
            t2 = v2;
            t3 = v3_;
        } else {
            T[0] = 0.0;
            SharedLog sl;
            sl.init(P, e, st, bin);
            for (int m = 1; m < P.n_mats; ++m) {
                const MatDesc& md = P.mats[m];
                T[m * kBlock] = md.has_tables ? sl.eval(P, md.mu, e, st, bin) : 0.0;
            }
        }
    }

    __device__ __forceinline__ double mu(const TransportParams& P, int code, float dens) const
    {
        if (FMT == kFmtP4) {
            if (REG) {
                const double lo = (code & 1) ? t1 : t0;
                const double hi = (code & 1) ? t3 : t2;
                return (code & 2) ? hi : lo;
            }
            return T[code * kBlock];
        }
        if (FMT == kFmtP8)
            return T[P.pal_mat[code] * kBlock] * (double)P.pal_dens[code];
        return T[code * kBlock] * (double)dens;
    }
};

// Voxel fetch: code (P4/P8 palette index or raw material id) + raw density.
template <int FMT>
__device__ __forceinline__ void fetch(const Grid& G, int ix, int iy, int iz, int& code, float& dens)
{
    const uint32_t c = brick_cell(G, ix, iy, iz);
    if (FMT == kFmtP4) {
        code = load_code_p4(G, c);
    } else if (FMT == kFmtP8) {
        code = load_code_p8(G, c);
    } else {
        code = __ldg(G.vox + c);
        dens = load_density_raw(G, c);
    }
}

template <int FMT>
__device__ __forceinline__ int material_of(const TransportParams& P, int code)
{
    return FMT == kFmtRaw ? code : P.pal_mat[code];
}

// Brick address split into per-axis terms (see brick_cell): cell = ax+ay+az,
// and a step only recomputes the term of the axis it crosses.
__device__ __forceinline__ uint32_t term_x(const Grid&, int i) { return ((uint32_t)(i >> 2) << 6) | (uint32_t)(i & 3); }
__device__ __forceinline__ uint32_t term_y(const Grid& G, int i)
{
    return (uint32_t)(i >> 2) * ((uint32_t)G.nbx << 6) + ((uint32_t)(i & 3) << 2);
}
__device__ __forceinline__ uint32_t term_z(const Grid& G, int i)
{
    return (uint32_t)(i >> 2) * ((uint32_t)G.nbx * (uint32_t)G.nby << 6) + ((uint32_t)(i & 3) << 4);
}

// Issue the load of a voxel; decoding is deferred to the step that uses it
// so the load latency overlaps a whole step.
template <int FMT>
__device__ __forceinline__ void prefetch(const Grid& G, uint32_t cell, uint32_t& raw, uint32_t& shift,
                                         float& dens)
{
    if (FMT == kFmtP4) {
        raw = (uint32_t)__ldg(G.vox + (cell >> 1)); // consumed one step later
        shift = (cell & 1u) << 2;
    } else {
        raw = __ldg(G.vox + cell);
        if (FMT == kFmtRaw)
            dens = load_density_raw(G, cell);
    }
}

template <int FMT>
__device__ __forceinline__ int decode(uint32_t raw, uint32_t shift)
{
    if (FMT == kFmtP4)
        return (int)((raw >> shift) & 0xFu);
    return (int)raw;
}

// ------------------------------------------------------------------ walker
struct Walk {
    double ox, oy, oz;    // ray origin
    double rx, ry, rz;    // ray direction
    double tnx, tny, tnz; // next boundary crossing per axis
    double dtx, dty, dtz; // per-voxel increments (march: dtx = step length)
    double t, texit, depth, target;
    double rdx, rdy, rdz; // 1 / dt per axis (macro-cell skips)
    int ix, iy, iz;       // current voxel (march: ix = sample j, iy = n samples)
    int sx, sy, sz;
    uint32_t ax, ay, az;  // per-axis brick address terms of the current voxel
    uint32_t raw;         // prefetched voxel (undecoded) ...
    uint32_t shift;       // ... and its nibble position (P4)
    float dens;
    double mu_hit;        // free path: mu of the voxel it ends in
    int march;
    int hit;
    uint32_t skipped;     // voxel visits integrated inside skipped macro cells
    uint32_t steps;       // loop iterations of this walk
};



template <int FMT, bool FAST>
__device__ __noinline__ bool walk_begin(const TransportParams& P, Walk& w, V3 o, V3 d,
                                           double target, bool march, DevStatus* st, int bin)
{
    double t0, t1;
    bool bad;
    w.ox = o.x;
    w.oy = o.y;
    w.oz = o.z;
    w.rx = d.x;
    w.ry = d.y;
    w.rz = d.z;
    w.hit = 0;
    w.depth = 0.0;
    w.steps = 0;
    w.skipped = 0;
    if (!clip_to_grid<FAST>(P.G, o, d, t0, t1, bad)) {
        if (bad)
            raise(st, XS_E_INVALID_ARGUMENT, 0, bin, 0.0, 0.0);
        return false;
    }
    w.target = target;
    w.texit = t1;
    w.t = t0;
    if (march) { // REF trace.cpp:116-134
        w.march = 1;
        const int n = (int)ceil((t1 - t0) / P.march_h);
        w.iy = n < 1 ? 1 : n;
        w.ix = 0;
        w.dtx = P.march_h;
        return true;
    }
    w.march = 0;
    const V3 p = o + d * t0;
    const Grid& G = P.G;
    start_axis<FAST>(p.x, o.x, d.x, G.ox, G.hx, G.ihx, G.nx, t0, w.ix, w.sx, w.tnx, w.dtx);
    start_axis<FAST>(p.y, o.y, d.y, G.oy, G.hy, G.ihy, G.ny, t0, w.iy, w.sy, w.tny, w.dty);
    start_axis<FAST>(p.z, o.z, d.z, G.oz, G.hz, G.ihz, G.nz, t0, w.iz, w.sz, w.tnz, w.dtz);
    w.ax = term_x(G, w.ix);
    w.ay = term_y(G, w.iy);
    w.az = term_z(G, w.iz);
    prefetch<FMT>(G, w.ax + w.ay + w.az, w.raw, w.shift, w.dens);
    // 1/dt estimates for macro-cell skips (cross_count corrects them exactly)
    w.rdx = fabs(d.x) * G.ihx;
    w.rdy = fabs(d.y) * G.ihy;
    w.rdz = fabs(d.z) * G.ihz;
    return true;
}

// Boundaries tn + j*dt (j = 0..k) with tn + j*dt <= tm: how many an axis
// crosses while the ray traverses a skipped macro cell (k = crossings left
// inside the cell along that axis; k + 1 means it also leaves the cell).
// Exact small-integer <-> double conversions on the fp64 pipe (fixed
// latency) instead of I2F/F2I.F64 (variable-latency MIO unit): 2^52 has an
// ulp of 1, so its bit pattern with k in the low word is 2^52 + k.
__device__ __forceinline__ double u2d_small(uint32_t k) // exact for any u32
{
    return __hiloint2double(0x43300000, (int)k) - 4503599627370496.0;
}
__device__ __forceinline__ int d2i_trunc_small(double x) // trunc(x) for 0 <= x < 2^31
{
    return __double2loint(__dadd_rz(x, 4503599627370496.0));
}

__device__ __forceinline__ int cross_count(double tn, double dt, double rdt, double tm, int k, int s)
{
    // Boundaries tn + j dt (j = 0..k) at or before tm.  Straight-line code
    // (estimate, then both one-step corrections evaluated together) so the
    // three axes overlap instead of running as three divergent branches.
    // k == 0 gives 1 when tn == tm (the plain Siddon crossing, REF
    // trace.cpp:146-153); axes without a crossing (s == 0 or tn > tm) give 0.
    int n = d2i_trunc_small((tm - tn) * rdt) + 1; // tm >= tn whenever the result is used
    n = n > k + 1 ? k + 1 : n;
    n = n < 1 ? 1 : n;
    const double lo = tn + u2d_small(n - 1) * dt; // boundary n-1 (must be <= tm)
    const double hi = tn + u2d_small(n) * dt;     // boundary n (must be > tm)
    n = lo > tm ? n - 1 : ((n <= k && hi <= tm) ? n + 1 : n);
    return (s != 0 && tn <= tm) ? (n < 1 ? 1 : n) : 0;
}

// Re-establish the exact walker at ray parameter t (REF start_walk,
// trace.cpp:72-103, applied at the exit of a skipped macro cell).  Returns
// false when the ray has left the grid.
__device__ __forceinline__ bool restart_axis(double p, double o, double d, double org, double hs,
                                             double inv_h, int n, double t, int step, double dt,
                                             int& idx, double& tn)
{
    idx = voxel_of(p, org, inv_h, n);
    if (step > 0)
        tn = (org + (idx + 1) * hs - o) / d;
    else if (step < 0)
        tn = (org + idx * hs - o) / d;
    else
        return true;
    while (tn <= t) {
        idx += step;
        tn += dt;
    }
    return idx >= 0 && idx < n;
}

// One voxel (REF trace.cpp:136-155 / :202-228).  Branch-free axis advance;
// the next voxel's load is issued before this step's fp64 chain and decoded
// only in the next step.
template <int FMT, bool REG, bool SKIP>
__device__ __forceinline__ bool walk_step(const TransportParams& P, const MuTab<FMT, REG>& tab,
                                          Walk& w)
{
    const Grid& G = P.G;
    if (w.march) { // REF trace.cpp:124-133
        const double ta = w.t + w.ix * w.dtx;
        const double tb = w.texit < ta + w.dtx ? w.texit : ta + w.dtx;
        const double tm = 0.5 * (ta + tb);
        const double px = w.ox + w.rx * tm, py = w.oy + w.ry * tm, pz = w.oz + w.rz * tm;
        int code;
        float dens = 0.f;
        fetch<FMT>(G, voxel_of(px, G.ox, G.ihx, G.nx), voxel_of(py, G.oy, G.ihy, G.ny),
                   voxel_of(pz, G.oz, G.ihz, G.nz), code, dens);
        w.depth += tab.mu(P, code & ~G.ubit, dens) * (tb - ta);
        return ++w.ix < w.iy;
    }
    const int code = decode<FMT>(w.raw, w.shift);
    if (SKIP) {
        // One step = up to the next boundary crossing, or, in a uniform 8^3
        // macro cell or 4^3 brick (code flags), up to its exit: k* boundaries of
        // each axis remain inside the cell (0 outside uniform cells, where
        // this is exactly REF's voxel step).  Branch-free, so lanes in
        // uniform and mixed cells do not diverge.
        const int c = code & ~G.ubit;
        // k* = boundaries left inside the uniform 8^3 cell / 4^3 brick (0 outside)
        const int um = (code & G.u8bit) ? 7 : ((code & G.u4bit) ? 3 : 0);
        const int kx = (w.sx > 0 ? ~w.ix : w.ix) & um;
        const int ky = (w.sy > 0 ? ~w.iy : w.iy) & um;
        const int kz = (w.sz > 0 ? ~w.iz : w.iz) & um;
        const double fx = w.tnx + u2d_small(kx) * w.dtx, fy = w.tny + u2d_small(ky) * w.dty,
                     fz = w.tnz + u2d_small(kz) * w.dtz;
        const double ex = kx ? fx : w.tnx;
        const double ey = ky ? fy : w.tny;
        const double ez = kz ? fz : w.tnz;
        double tm = ex;
        if (ey < tm)
            tm = ey;
        if (ez < tm)
            tm = ez;
        if (w.texit < tm)
            tm = w.texit;
        const double mu = tab.mu(P, c, w.dens);
        const double seg = mu * (tm - w.t);
        const double nd = w.depth + seg;
        if (nd >= w.target) { // free path ends in this voxel / cell; t_hit in hit_t()
            w.hit = 1;
            w.mu_hit = mu;
            w.texit = tm;
            return false;
        }
        const int nx = cross_count(w.tnx, w.dtx, w.rdx, tm, kx, w.sx);
        const int ny = cross_count(w.tny, w.dty, w.rdy, tm, ky, w.sy);
        const int nz = cross_count(w.tnz, w.dtz, w.rdz, tm, kz, w.sz);
        const int nix = w.ix + nx * w.sx, niy = w.iy + ny * w.sy, niz = w.iz + nz * w.sz;
        const bool inside = (tm < w.texit) && (uint32_t)nix < (uint32_t)G.nx &&
                            (uint32_t)niy < (uint32_t)G.ny && (uint32_t)niz < (uint32_t)G.nz;
        const uint32_t nax = nx ? term_x(G, nix) : w.ax;
        const uint32_t nay = ny ? term_y(G, niy) : w.ay;
        const uint32_t naz = nz ? term_z(G, niz) : w.az;
        if (inside)
            prefetch<FMT>(G, nax + nay + naz, w.raw, w.shift, w.dens);
        w.depth = nd;
        w.t = tm;
        w.tnx = nx ? w.tnx + u2d_small(nx) * w.dtx : w.tnx;
        w.tny = ny ? w.tny + u2d_small(ny) * w.dty : w.tny;
        w.tnz = nz ? w.tnz + u2d_small(nz) * w.dtz : w.tnz;
        if (um)
            w.skipped += (uint32_t)(nx + ny + nz) - 1u;
        w.ix = nix;
        w.iy = niy;
        w.iz = niz;
        w.ax = nax;
        w.ay = nay;
        w.az = naz;
        return inside;
    }
    const float dens = w.dens;
    double tn = w.tnx;
    if (w.tny < tn)
        tn = w.tny;
    if (w.tnz < tn)
        tn = w.tnz;
    if (w.texit < tn)
        tn = w.texit;
    const bool cx = w.tnx == tn, cy = w.tny == tn, cz = w.tnz == tn;
    const int nix = cx ? w.ix + w.sx : w.ix;
    const int niy = cy ? w.iy + w.sy : w.iy;
    const int niz = cz ? w.iz + w.sz : w.iz;
    const bool inside = (tn < w.texit) && (uint32_t)nix < (uint32_t)G.nx &&
                        (uint32_t)niy < (uint32_t)G.ny && (uint32_t)niz < (uint32_t)G.nz;
    const uint32_t nax = cx ? term_x(G, nix) : w.ax;
    const uint32_t nay = cy ? term_y(G, niy) : w.ay;
    const uint32_t naz = cz ? term_z(G, niz) : w.az;
    if (inside)
        prefetch<FMT>(G, nax + nay + naz, w.raw, w.shift, w.dens);

    const double mu = tab.mu(P, code & ~G.ubit, dens);
    const double seg = mu * (tn - w.t);
    const double nd = w.depth + seg;
    if (nd >= w.target) { // free path ends inside this voxel; t_hit in hit_t()
        w.hit = 1;
        w.mu_hit = mu;
        w.texit = tn;
        return false;
    }
    w.depth = nd;
    w.t = tn;
    w.tnx = cx ? w.tnx + w.dtx : w.tnx;
    w.tny = cy ? w.tny + w.dty : w.tny;
    w.tnz = cz ? w.tnz + w.dtz : w.tnz;
    w.ix = nix;
    w.iy = niy;
    w.iz = niz;
    w.ax = nax;
    w.ay = nay;
    w.az = naz;
    return inside;
}

// REF trace.cpp:212-213: the interaction point's ray parameter.
__device__ __forceinline__ double hit_t(const Walk& w)
{
    return (w.mu_hit > 0.0) ? w.t + (w.target - w.depth) / w.mu_hit : w.texit;
}

// ------------------------------------------------------ shared accumulators
__device__ __forceinline__ void sadd(unsigned long long* p, uint64_t v)
{
    if (v)
        atomicAdd(p, (unsigned long long)v);
}

__device__ __forceinline__ bool tally_limbs(unsigned long long* slot, double x, int log2_unit)
{
    uint64_t l0, l1, l2;
    if (!quantize(ldexp(x, -log2_unit), l0, l1, l2))
        return false;
    sadd(slot + 0, l0);
    sadd(slot + 1, l1);
    sadd(slot + 2, l2);
    return true;
}

struct Block {
    unsigned long long* bins;   // n_bins * 8
    unsigned long long* ledger; // 24
    unsigned long long* diag;   // 8
};

__device__ __forceinline__ void ledger_add(const TransportParams& P, const Block& B, int k,
                                           double w, DevStatus* st, int bin)
{
    if (w != 0.0 && !tally_limbs(B.ledger + 4 * k, w, P.log2_w))
        raise(st, XS_E_RUNTIME, kErrTallyOverflow, bin, 0.0, w);
}

// Scoring task: pixel << 6 | slot (n_pixels < 2^26, checked on the host).
// The scoring FIFO has qlen = H * splitting + 1 entries and its tail wraps
// (atomicInc), so it can never fill; the free-path FIFO follows it.
__device__ __forceinline__ void push_score(WarpHdr* hdr, uint32_t* q, uint32_t qlen, int s, uint32_t pixel)
{
    const uint32_t i = atomicInc(&hdr->tail, qlen - 1u);
    q[i] = pixel << 6 | (uint32_t)s;
}

__device__ __forceinline__ void push_free(WarpHdr* hdr, uint32_t* q, uint32_t qlen, int s)
{
    const uint32_t i = atomicAdd(&hdr->ftail, 1u);
    q[qlen + (i & (kFreeQ - 1))] = (uint32_t)s;
}


// History end (REF run_history :225-241): bin statistics from the exact
// fixed-point history total, per-pixel grouping for the variance, free slot.
__device__ __noinline__ void finalize_history(const TransportParams& P, const Block& B, Slot* slots,
                                              WarpHdr* hdr, int s, uint64_t var_base, DevStatus* st)
{
    Slot& S = slots[s];
    const double t = dequantize(S.T[0], S.T[1], S.T[2], P.log2_img);
    unsigned long long* bs = B.bins + 8 * S.bin;
    if (t != 0.0) {
        if (!tally_limbs(bs, t, P.log2_img) || !tally_limbs(bs + 3, t * t, 2 * P.log2_img))
            raise(st, XS_E_RUNTIME, kErrTallyOverflow, S.bin, S.E, t);
    }
    if (P.track_var) {
        const uint32_t* vp = P.var_pix + var_base;
        const double* vv = P.var_val + var_base;
        const int n = S.n_var < P.var_cap ? S.n_var : P.var_cap;
        for (int a = 0; a < n; ++a) {
            const uint32_t pa = vp[a];
            bool dup = false;
            for (int b = 0; b < a; ++b)
                if (vp[b] == pa) {
                    dup = true;
                    break;
                }
            if (dup)
                continue;
            double c = vv[a];
            for (int b = a + 1; b < n; ++b)
                if (vp[b] == pa)
                    c += vv[b];
            if (!tally_global(P.accum + P.off_var + 4ull * pa, c * c, 2 * P.log2_img))
                raise(st, XS_E_RUNTIME, kErrTallyOverflow, S.bin, S.E, c);
        }
    }
    sadd(B.diag + 2, 1);
    atomicOr(&hdr->free_mask, 1ull << s);
}

__device__ __forceinline__ void end_history(const TransportParams& P, const Block& B, Slot* slots,
                                            WarpHdr* hdr, int s, uint64_t var_base, DevStatus* st)
{
    __threadfence_block(); // this lane's tallies / scratch before the hand-off
    if (atomicSub(&slots[s].pending, 1) == 1)
        finalize_history(P, B, slots, hdr, s, var_base, st);
}

// Free-path completion: the reference's per-history event logic
// (run_history :141-223) on the history's own Philox stream.
template <int FMT>
__device__ __noinline__ void history_event(const TransportParams& P, const Block& B, Slot* slots,
                                           WarpHdr* hdr, uint32_t* q, uint32_t qlen, int s,
                                           bool hit, double t_hit, int vix, int viy, int viz,
                                           uint64_t var_base, DevStatus* st)
{
    Slot& S = slots[s];
    const int bin = S.bin;
    const double W = S.W;
    if (!hit) {
        ledger_add(P, B, 1, W, st, bin);
        end_history(P, B, slots, hdr, s, var_base, st);
        return;
    }
    const V3 dir = v3(S.dx, S.dy, S.dz);
    const V3 pos = v3(S.px, S.py, S.pz) + dir * t_hit;
    int code;
    float dens;
    fetch<FMT>(P.G, vix, viy, viz, code, dens);
    const int mat = material_of<FMT>(P, code & ~P.G.ubit);
    const MatDesc& md = P.mats[mat];
    const double E = S.E;
    // select_interaction (cross_sections.cpp:81-96)
    const double pe = loglog_or_fail(P, md.pe, E, st, bin);
    const double incoh = loglog_or_fail(P, md.incoh, E, st, bin);
    const double coh = loglog_or_fail(P, md.coh, E, st, bin);
    const double total = pe + incoh + coh;
    if (!(total > 0.0))
        raise(st, XS_E_RUNTIME, kErrSigmaAll, bin, E, (double)mat);
    const double u = slot_uniform(&S, P.k0, P.k1, P.angle) * total;
    const int kind = u < pe ? K_PE : (u < pe + incoh ? K_COMPTON : K_RAYLEIGH);
    if (kind == K_PE) {
        ledger_add(P, B, 2, W, st, bin);
        end_history(P, B, slots, hdr, s, var_base, st);
        return;
    }
    S.px = pos.x;
    S.py = pos.y;
    S.pz = pos.z;
    S.ix = dir.x;
    S.iy = dir.y;
    S.iz = dir.z;
    S.e_in = E;
    S.kind = kind;
    S.mat = mat;
    S.w_split = W / P.splitting;
    { // the cross-section prefactor of p_lambda is the same for all its rays
        const double sigma = (kind == K_COMPTON ? incoh : coh) * kBarn;
        if (!(sigma > 0.0))
            raise(st, XS_E_RUNTIME, kind == K_COMPTON ? kErrSigmaIncoh : kErrSigmaCoh, bin, E, 0.0);
        const double r0 = kR0;
        S.pref = kPi * r0 * r0 / sigma;
    }
    atomicAdd(&S.pending, P.splitting);
#pragma unroll 1
    for (int k = 0; k < P.splitting; ++k) { // REF :162-164 pixel draws
        int iu = (int)(slot_uniform(&S, P.k0, P.k1, P.angle) * P.nu);
        int iv = (int)(slot_uniform(&S, P.k0, P.k1, P.angle) * P.nv);
        iu = iu < P.nu - 1 ? iu : P.nu - 1;
        iv = iv < P.nv - 1 ? iv : P.nv - 1;
        push_score(hdr, q, qlen, s, (uint32_t)(iv * P.nu + iu));
    }
    // continuation (REF :195-205)
    V3 ndir;
    double nE = E;
    if (kind == K_COMPTON) { // samplers.cpp:32-52
        const double alpha = E / kMec2;
        const double q_max = momentum_transfer(E, kPi);
        const double s_max = form_S(P, md, q_max);
        double theta = 0.0, ap = 0.0, phi = 0.0;
        if (!(s_max > 0.0)) {
            raise(st, XS_E_RUNTIME, kErrComptonS, bin, E, 0.0);
        } else {
            for (;;) {
                const double t = 1.0 + 2.0 * alpha; // kahn_sample_cos_theta, samplers.cpp:12-30
                double cos_th;
                for (;;) {
                    const double r1 = slot_uniform(&S, P.k0, P.k1, P.angle);
                    const double r2 = slot_uniform(&S, P.k0, P.k1, P.angle);
                    const double r3 = slot_uniform(&S, P.k0, P.k1, P.angle);
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
                theta = nl_acos(cc);
                const double sv = form_S(P, md, momentum_transfer(E, theta));
                if (slot_uniform(&S, P.k0, P.k1, P.angle) * s_max <= sv) {
                    ap = alpha / (1.0 + alpha * (1.0 - nl_cos(theta)));
                    phi = 2.0 * kPi * slot_uniform(&S, P.k0, P.k1, P.angle);
                    break;
                }
            }
        }
        ndir = rotate_direction(dir, theta, phi);
        nE = ap * kMec2;
    } else { // samplers.cpp:106-125
        const double q_max = momentum_transfer(E, kPi);
        const double tot = cumulative_mass(P, md, q_max);
        double theta = 0.0, phi = 0.0;
        if (!(tot > 0.0)) {
            raise(st, XS_E_RUNTIME, kErrRayleighF, bin, E, 0.0);
        } else {
            const double scale = kHc / E;
            for (;;) {
                const double qq = invert_mass(P, md, slot_uniform(&S, P.k0, P.k1, P.angle) * tot, q_max);
                const double sh = 1.0 < qq * scale ? 1.0 : qq * scale;
                const double cos_th = 1.0 - 2.0 * sh * sh;
                if (slot_uniform(&S, P.k0, P.k1, P.angle) * 2.0 <= 1.0 + cos_th * cos_th) {
                    const double cc = cos_th < -1.0 ? -1.0 : (1.0 < cos_th ? 1.0 : cos_th);
                    theta = nl_acos(cc);
                    phi = 2.0 * kPi * slot_uniform(&S, P.k0, P.k1, P.angle);
                    break;
                }
            }
        }
        ndir = rotate_direction(dir, theta, phi);
    }
    S.dx = ndir.x;
    S.dy = ndir.y;
    S.dz = ndir.z;
    S.E = nE;
    const int gen = ++S.gen;
    bool alive = true;
    double Wn = W;
    if (gen >= P.max_inter) { // REF :207-211
        ledger_add(P, B, 3, W, st, bin);
        alive = false;
    } else if (S.wmin > 0.0 && W < S.wmin) { // REF :213-222
        if (slot_uniform(&S, P.k0, P.k1, P.angle) < P.survival) {
            const double boosted = W / P.survival;
            ledger_add(P, B, 5, boosted - W, st, bin);
            Wn = boosted;
        } else {
            ledger_add(P, B, 4, W, st, bin);
            alive = false;
        }
    }
    if (alive) {
        S.W = Wn;
        S.target = -nl_log(slot_uniform(&S, P.k0, P.k1, P.angle));
        push_free(hdr, q, qlen, s);
    } else {
        end_history(P, B, slots, hdr, s, var_base, st);
    }
}

// History start (REF run_history :120-138, sample_emission :73-87).
__device__ __noinline__ void history_start(const TransportParams& P, const Block& B, Slot* slots,
                                           WarpHdr* hdr, uint32_t* q, uint32_t qlen,
                                           const uint64_t* sstart, int s, uint64_t h, DevStatus* st)
{
    Slot& S = slots[s];
    int lo = 0, hi = P.n_bins; // last bin b with start[b] <= h (skips empty bins)
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (sstart[mid] <= h)
            lo = mid;
        else
            hi = mid;
    }
    const int bin = lo;
    S.r_photon = (uint32_t)(h - sstart[lo]);
    S.r_bin = (uint32_t)lo;
    S.r_block = 0;
    S.r_pos = 4;
    const double u1 = slot_uniform(&S, P.k0, P.k1, P.angle);
    const double u2 = slot_uniform(&S, P.k0, P.k1, P.angle);
    const double xu = (u1 - 0.5) * P.nu * P.pitch;
    const double xv = (u2 - 0.5) * P.nv * P.pitch;
    const V3 c = v3(P.center[0], P.center[1], P.center[2]);
    const V3 ua = v3(P.uaxis[0], P.uaxis[1], P.uaxis[2]);
    const V3 target = (c + ua * xu) + v3(0.0, 0.0, 1.0) * xv;
    const V3 src = v3(P.src[0], P.src[1], P.src[2]);
    const V3 delta = target - src;
    const double d2 = dot(delta, delta);
    const V3 dir = delta / sqrt(d2);
    const double cos_psi = -dot(dir, v3(P.normal[0], P.normal[1], P.normal[2]));
    const double em_weight = P.det_area * cos_psi / d2;
    const double w0 = __ldg(P.bin_weight + bin) * em_weight / (double)__ldg(P.bin_count + bin);
    S.px = src.x;
    S.py = src.y;
    S.pz = src.z;
    S.dx = dir.x;
    S.dy = dir.y;
    S.dz = dir.z;
    S.E = __ldg(P.bin_energy + bin);
    S.W = w0;
    S.wmin = P.wmin_rel * w0;
    S.T[0] = S.T[1] = S.T[2] = 0ull;
    S.bin = bin;
    S.gen = 0;
    S.pending = 1;
    S.n_var = 0;
    ledger_add(P, B, 0, w0, st, bin);
    S.target = -nl_log(slot_uniform(&S, P.k0, P.k1, P.angle));
    push_free(hdr, q, qlen, s);
    atomicAnd(&hdr->free_mask, ~(1ull << s));
}

// Scoring-ray set-up (REF run_history :166-183): geometry, p(theta), e_out,
// response; returns the score prefactor (point_detector_score without exp(-tau)).
__device__ __noinline__ double score_setup(const TransportParams& P, const Slot& S, uint32_t pix,
                                              V3& o, V3& to_det, double& e_out, DevStatus* st)
{
    const int iu = (int)(pix % (uint32_t)P.nu);
    const int iv = (int)(pix / (uint32_t)P.nu);
    const double du = (iu + 0.5 - 0.5 * P.nu) * P.pitch;
    const double dv = (iv + 0.5 - 0.5 * P.nv) * P.pitch;
    const V3 c = v3(P.center[0], P.center[1], P.center[2]);
    const V3 ua = v3(P.uaxis[0], P.uaxis[1], P.uaxis[2]);
    const V3 px = (c + ua * du) + v3(0.0, 0.0, 1.0) * dv;
    o = v3(S.px, S.py, S.pz); // the interaction point until the next free path ends
    const V3 delta = px - o;
    const double d2 = dot(delta, delta);
    to_det = delta / sqrt(d2);
    double cos_t = dot(v3(S.ix, S.iy, S.iz), to_det);
    cos_t = cos_t < -1.0 ? -1.0 : (1.0 < cos_t ? 1.0 : cos_t);
    const double theta = nl_acos(cos_t);
    const MatDesc& md = P.mats[S.mat];
    const double E = S.e_in;
    double p_dir;
    if (S.kind == K_COMPTON) { // cross_sections.cpp:56-66 (ratio shared by kn_core and e_out)
        const double ratio = compton_ratio(E, theta);
        const double s = nl_sin(theta);
        const double kn = ratio * ratio * (ratio + 1.0 / ratio - s * s);
        p_dir = S.pref * kn * form_S(P, md, momentum_transfer(E, theta));
        e_out = E * ratio;
    } else { // cross_sections.cpp:68-79
        const double c2 = nl_cos(theta);
        const double f = form_F(P, md, momentum_transfer(E, theta));
        p_dir = S.pref * (1.0 + c2 * c2) * f * f;
        e_out = E;
    }
    double dep = 0.0;
    if (!tab_linear(mtab(P, P.resp_deposit), e_out, dep))
        raise(st, XS_E_OUT_OF_RANGE, kErrTableRange, S.bin, e_out, 1.0);
    return dep / e_out * p_dir * S.w_split * P.n_pixels / (2.0 * kPi * d2);
}

} // namespace

// per-warp shared memory: slots, header, scoring + free-path FIFOs (8-aligned)
__host__ __device__ inline size_t warp_bytes_of(int H, int qlen)
{
    return ((size_t)H * sizeof(Slot) + sizeof(WarpHdr) + (size_t)(qlen + kFreeQ) * 4 + 7) & ~(size_t)7;
}

// =================================================================== kernel
template <int FMT, bool REG, bool SKIP>
__global__ void __launch_bounds__(kBlock, XSD_MIN_BLOCKS) transport_kernel(const __grid_constant__ TransportParams P)
{
    extern __shared__ __align__(16) unsigned char smem[];
    const int H = P.slots_per_warp;
    const uint32_t qlen = (uint32_t)P.queue_len; // H * splitting + 1
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const unsigned lt_mask = (1u << lane) - 1u;

    // ---- carve shared memory
    Block B;
    B.bins = reinterpret_cast<unsigned long long*>(smem);
    B.ledger = B.bins + 8 * P.n_bins;
    B.diag = B.ledger + 24;
    uint64_t* sstart = reinterpret_cast<uint64_t*>(B.diag + 8);
    unsigned char* p = reinterpret_cast<unsigned char*>(sstart + P.n_bins + 1);
    const size_t warp_bytes = warp_bytes_of(H, P.queue_len);
    unsigned char* wbase = p + (size_t)warp * warp_bytes;
    Slot* slots = reinterpret_cast<Slot*>(wbase);
    WarpHdr* hdr = reinterpret_cast<WarpHdr*>(wbase + (size_t)H * sizeof(Slot));
    uint32_t* q = reinterpret_cast<uint32_t*>(hdr + 1);
    MuTab<FMT, REG> tab;
    tab.T = reinterpret_cast<double*>(p + (size_t)kWarps * warp_bytes) + threadIdx.x;
    tab.energy = -1.0;

    for (int i = threadIdx.x; i < 8 * P.n_bins + 32; i += blockDim.x)
        B.bins[i] = 0ull;
    for (int i = threadIdx.x; i <= P.n_bins; i += blockDim.x)
        sstart[i] = P.bin_start[i];
    const unsigned long long all_free = H >= 64 ? ~0ull : ((1ull << H) - 1ull);
    if (lane == 0) {
        hdr->tail = 0;
        hdr->ftail = 0;
        hdr->free_mask = all_free;
    }
    __syncthreads();

    DevStatus* st = P.status;
    const uint64_t gwarp = (uint64_t)blockIdx.x * kWarps + warp;
    const bool march = P.step_voxels > 1;

    uint32_t head = 0, fhead = 0;     // warp-uniform FIFO heads
    uint64_t wq_next = 0, wq_end = 0; // warp-uniform history reservation
    bool pool_empty = false;
    uint32_t c_fp = 0, c_sc = 0, c_rays = 0, c_int = 0, c_iter = 0, c_wit = 0;

    // Each iteration: admit histories, set up one ray per lane from the FIFO,
    // walk until every lane's ray has ended, process the 32 completions.
    // The walker state is local to an iteration, so nothing of it is live
    // across the out-of-line event calls (no ABI save/restore traffic).
    for (;;) {
        // ------------------------------------------------ 1. admit histories
        const unsigned long long free_now = hdr->free_mask;
        if (free_now && !pool_empty) {
            const int n_free = __popcll(free_now);
            int n_new = 0;
            uint64_t first = 0;
            while (n_new == 0 && !pool_empty) {
                if (wq_next >= wq_end) {
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
                        break;
                    }
                }
                const uint64_t avail = wq_end - wq_next;
                n_new = (uint64_t)n_free < avail ? n_free : (int)avail;
                if (n_new > 32)
                    n_new = 32;
                first = wq_next;
                wq_next += n_new;
            }
            if (lane < n_new) {
                unsigned long long m = free_now; // lane-th set bit
                for (int k = 0; k < lane; ++k)
                    m &= m - 1;
                const int s = __ffsll((long long)m) - 1;
                history_start(P, B, slots, hdr, q, qlen, sstart, s, first + lane, st);
            }
        }
        __syncwarp();

        // ------------------------------------------------ 2. pop + set up
        const uint32_t tail = *(volatile uint32_t*)&hdr->tail;
        const uint32_t ftail = *(volatile uint32_t*)&hdr->ftail;
        const uint32_t avail = tail >= head ? tail - head : tail + qlen - head;
        const uint32_t n_s = avail < 32u ? avail : 32u;
        const uint32_t favail = ftail - fhead;
        const uint32_t n_f = favail < 32u - n_s ? favail : 32u - n_s;
        int ttype = T_NONE, tslot = 0;
        uint32_t tpix = 0;
        double tpre = 0.0;
        bool walking = false;
        Walk w;
        w.march = 0;
        w.hit = 0;
        w.steps = 0;
        w.skipped = 0;
        w.depth = 0.0;
        if ((uint32_t)lane < n_s + n_f) {
            uint32_t task;
            if ((uint32_t)lane < n_s) {
                uint32_t i = head + lane;
                task = q[i >= qlen ? i - qlen : i];
                ttype = T_SCORE;
            } else {
                task = q[qlen + ((fhead + lane - n_s) & (kFreeQ - 1))];
                ttype = T_FREE;
            }
            tslot = (int)(task & 63u);
            tpix = task >> 6;
            const Slot& S = slots[tslot];
            if (ttype == T_FREE) { // REF trace.cpp:189-230
                if (tab.energy != S.E)
                    tab.fill(P, S.E, st, S.bin);
                walking = walk_begin<FMT, SKIP>(P, w, v3(S.px, S.py, S.pz), v3(S.dx, S.dy, S.dz), S.target,
                                          false, st, S.bin);
            } else {
                V3 o, to_det;
                double e_out;
                tpre = score_setup(P, S, tpix, o, to_det, e_out, st);
                if (tab.energy != e_out) // REF trace_attenuation builds MuField(e_out)
                    tab.fill(P, e_out, st, S.bin);
                walking = walk_begin<FMT, SKIP>(P, w, o, to_det, CUDART_INF, march, st, S.bin);
                ++c_rays;
            }
        }
        head += n_s;
        head = head >= qlen ? head - qlen : head;
        fhead += n_f;

        // ------------------------------------------------ termination
        if (__ballot_sync(kFull, ttype != T_NONE) == 0) {
            if (pool_empty && tail == head && ftail == fhead && hdr->free_mask == all_free)
                break;
            if (*(volatile int32_t*)&st->code != 0)
                break;
            continue;
        }

        // ------------------------------------------------ 3. walk in lockstep
        while (__ballot_sync(kFull, walking)) {
            ++c_wit;
            if (walking) {
                walking = walk_step<FMT, REG, SKIP>(P, tab, w);
                ++w.steps;
            }
        }

        // ------------------------------------------------ 4. completions
        if (ttype != T_NONE) {
            if (ttype == T_FREE)
                c_fp += w.steps + w.skipped;
            else
                c_sc += w.steps + w.skipped;
            c_iter += w.steps;
            const uint64_t var_base = (gwarp * H + tslot) * (uint64_t)P.var_cap;
            if (ttype == T_SCORE) { // REF run_history :178-193
                Slot& S = slots[tslot];
                const double x = tpre * nl_exp(-w.depth);
                uint64_t l0 = 0, l1 = 0, l2 = 0;
                if (!isfinite(x)) {
                    raise(st, XS_E_RUNTIME, kErrNonFinite, S.bin, S.e_in, x);
                } else if (!quantize(ldexp(x, -P.log2_img), l0, l1, l2)) {
                    raise(st, XS_E_RUNTIME, kErrTallyOverflow, S.bin, S.e_in, x);
                } else {
                    unsigned long long* img = P.accum + P.off_image + 4ull * tpix;
                    red_add(img + 0, l0);
                    red_add(img + 1, l1);
                    red_add(img + 2, l2);
                    sadd(&S.T[0], l0);
                    sadd(&S.T[1], l1);
                    sadd(&S.T[2], l2);
                }
                if (P.track_var) {
                    const int k = atomicAdd(&S.n_var, 1);
                    if (k < P.var_cap) {
                        P.var_pix[var_base + k] = tpix;
                        P.var_val[var_base + k] = x;
                    }
                }
                end_history(P, B, slots, hdr, tslot, var_base, st);
            } else {
                const bool hit = w.hit != 0;
                if (hit)
                    ++c_int;
                history_event<FMT>(P, B, slots, hdr, q, qlen, tslot, hit, hit ? hit_t(w) : 0.0, w.ix,
                                   w.iy, w.iz, var_base, st);
            }
        }
        __syncwarp();
        if (*(volatile int32_t*)&st->code != 0)
            break;
    }

    // flush this warp's counters and the block's statistics
    sadd(B.diag + 0, c_fp);
    sadd(B.diag + 1, c_sc);
    sadd(B.diag + 3, c_rays);
    sadd(B.diag + 4, c_int);
    sadd(B.diag + 5, c_iter);
    if (lane == 0)
        sadd(B.diag + 6, 32ull * c_wit);
    __syncthreads();
    for (int i = threadIdx.x; i < 8 * P.n_bins; i += blockDim.x)
        red_add(P.accum + P.off_bins + i, B.bins[i]);
    for (int i = threadIdx.x; i < 24; i += blockDim.x)
        red_add(P.accum + P.off_ledger + i, B.ledger[i]);
    for (int i = threadIdx.x; i < 8; i += blockDim.x)
        red_add(P.accum + P.off_diag + i, B.diag[i]);
}

// ----------------------------------------------------------------- launchers
static bool use_reg(const TransportParams& P) { return P.G.fmt == kFmtP4 && P.n_pal <= 4; }

size_t transport_smem_bytes(const TransportParams& P)
{
    const size_t warp_bytes = warp_bytes_of(P.slots_per_warp, P.queue_len);
    const int n_tab = P.G.fmt == kFmtP4 ? P.n_pal : P.n_mats;
    return (size_t)(8 * P.n_bins + 32) * 8 + (size_t)(P.n_bins + 1) * 8 + kWarps * warp_bytes +
           (use_reg(P) ? 0 : (size_t)n_tab * kBlock * 8);
}

int transport_block_size() { return kBlock; }

// Live histories per warp: as many as fit a shared-memory budget per block
// (the rest of the SM's 256 KB stays L1 for the stack frames and voxels).
int transport_pick_slots(TransportParams& P, int max_slots, size_t budget)
{
    int H = max_slots < 64 ? max_slots : 64;
    for (; H > 1; --H) {
        P.slots_per_warp = H;
        P.queue_len = H * P.splitting + 1;
        if (transport_smem_bytes(P) <= budget)
            break;
    }
    P.slots_per_warp = H;
    P.queue_len = H * P.splitting + 1;
    return H;
}

typedef void (*TransportFn)(const TransportParams);

static TransportFn kernel_for(const TransportParams& P)
{
    const bool skip = P.skip != 0 && P.G.ubit != 0;
    if (P.G.fmt == kFmtP4) {
        if (use_reg(P))
            return skip ? transport_kernel<kFmtP4, true, true> : transport_kernel<kFmtP4, true, false>;
        return skip ? transport_kernel<kFmtP4, false, true> : transport_kernel<kFmtP4, false, false>;
    }
    if (P.G.fmt == kFmtP8)
        return skip ? transport_kernel<kFmtP8, false, true> : transport_kernel<kFmtP8, false, false>;
    return transport_kernel<kFmtRaw, false, false>;
}

cudaError_t transport_prepare(const TransportParams& P, size_t smem, int* blocks_per_sm)
{
    const void* k = (const void*)kernel_for(P);
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess)
        return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, k, kBlock, smem);
}

cudaError_t launch_transport(const TransportParams& P, int grid, size_t smem, cudaStream_t s)
{
    kernel_for(P)<<<grid, kBlock, smem, s>>>(P);
    return cudaGetLastError();
}

} // namespace xsd
