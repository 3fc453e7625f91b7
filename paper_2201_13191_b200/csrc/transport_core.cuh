// transport_core.cuh — device building blocks shared by the two transport
// engines (transport.cu: persistent megakernel with per-warp shared-memory
// queues; wavefront.cu: kernel-per-stage pipeline with global queues).
//
// History state (Slot), the Philox stream, the mu tables, the Siddon walker
// (REF trace.cpp) and REF's per-history event logic (REF transport.cpp:114-243)
// live here.  The event logic is templated on a queue policy Q providing
//   Slot& slot(s); reserve_scores(n) -> base; push_score(base + k, s, pixel);
//   push_free(s); claim(s); release(s); fence()
// so both engines run the identical arithmetic per history.
#pragma once
#include <cmath>
#include <cstddef>

#include "physics.cuh"

namespace xsd {

namespace {

constexpr int kBlock = 128; // threads per block of every transport kernel (mu-table stride)

constexpr unsigned kFull = 0xffffffffu;
enum : int { T_NONE = -1, T_FREE = 0, T_SCORE = 1 };
enum : int { K_NONE = -1, K_PE = 0, K_COMPTON = 1, K_RAYLEIGH = 2 };

// ------------------------------------------------------------ smem layout
// A history's Philox stream (REF rng.hpp:11-67): counter {block, photon, bin,
// angle}, the current 4-word block and the read position in it.
struct SlotRng {
    uint32_t photon, bin, block, pos, b0, b1, b2, b3;
};

struct __align__(16) Slot { // (16: the wavefront admission writes it with 16-byte stores)
    double px, py, pz, dx, dy, dz; // photon position (= last interaction point) / direction
    double E, W, wmin, target;     // energy, weight, roulette floor, -ln u of the pending free path
    double ix, iy, iz;             // incoming direction at it
    double e_in, w_split;          // energy at it, weight per pseudo-particle
    double pref;                   // pi r0^2 / sigma(E) of its kind (REF cross_sections.cpp:56-79)
    unsigned long long T[3];       // history total, fixed-point limbs (unit U_img)
    SlotRng rng;                   // Philox stream
    int32_t bin, gen, kind, mat;
    int32_t pending;               // queued/in-flight scoring rays + 1 while alive
    int32_t n_var;                 // variance scratch entries
};

static_assert(sizeof(Slot) == 208 && offsetof(Slot, T) == 128 && offsetof(Slot, rng) == 152 &&
                  offsetof(Slot, bin) == 184 && offsetof(Slot, pending) == 200,
              "history_start's 16-byte stores assume this Slot layout");

// Philox4x32-10 block for counter {block, photon, bin, angle} and key
// {k0, k1} (REF rng.hpp:29-60).
__device__ __forceinline__ void philox_block(uint32_t block, uint32_t photon, uint32_t bin, uint32_t angle,
                                             uint32_t k0, uint32_t k1, uint32_t& o0, uint32_t& o1,
                                             uint32_t& o2, uint32_t& o3)
{
    uint32_t c0 = block, c1 = photon, c2 = bin, c3 = angle;
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
    o0 = c0;
    o1 = c1;
    o2 = c2;
    o3 = c3;
}

// REF Rng::uniform: the top 53 bits of a 64-bit word pair, centred.
__device__ __forceinline__ double words_to_uniform(uint32_t hi, uint32_t lo)
{
    const uint64_t bits = (((uint64_t)hi << 32) | lo) >> 11;
    return ((double)bits + 0.5) * 0x1p-53;
}

// The 10-round Philox block, out of line with scalar arguments and a uint4
// result (registers only): one copy serves every draw site of the event
// code, and the caller's stream state stays in registers.
__device__ __noinline__ uint4 philox_out(uint32_t block, uint32_t photon, uint32_t bin, uint32_t angle, uint32_t k0,
                                         uint32_t k1)
{
    uint4 o;
    philox_block(block, photon, bin, angle, k0, k1, o.x, o.y, o.z, o.w);
    return o;
}

// One Philox draw on a history's stream (REF rng.hpp:29-60).  The event code
// works on a local copy of the slot's stream (one load and one store per
// event instead of a slot round trip per draw).
__device__ __forceinline__ double slot_uniform(SlotRng* s, uint32_t k0, uint32_t k1, uint32_t angle)
{
    if (s->pos == 4) {
        const uint4 o = philox_out(s->block, s->photon, s->bin, angle, k0, k1);
        s->b0 = o.x;
        s->b1 = o.y;
        s->b2 = o.z;
        s->b3 = o.w;
        s->pos = 0;
        ++s->block;
    }
    const uint32_t hi = s->pos == 0 ? s->b0 : s->b2;
    const uint32_t lo = s->pos == 0 ? s->b1 : s->b3;
    s->pos += 2;
    return words_to_uniform(hi, lo);
}

// The j-th draw after stream state `r` without drawing the ones before it
// (Philox is counter-based): the wavefront engine draws a history's scoring
// pixels in parallel, one thread per ray, bit for bit REF's sequential order.
__device__ __forceinline__ double rng_uniform_at(const SlotRng& r, uint32_t j, uint32_t k0, uint32_t k1,
                                                 uint32_t angle)
{
    const uint32_t m0 = (4u - r.pos) >> 1; // draws left in the buffered block
    if (j < m0) {
        const uint32_t q = r.pos + 2 * j;
        return words_to_uniform(q == 0 ? r.b0 : r.b2, q == 0 ? r.b1 : r.b3);
    }
    const uint32_t k = j - m0;
    uint32_t o0, o1, o2, o3;
    philox_block(r.block + (k >> 1), r.photon, r.bin, angle, k0, k1, o0, o1, o2, o3);
    return (k & 1) ? words_to_uniform(o2, o3) : words_to_uniform(o0, o1);
}

// Draws j and j + 1 (a scoring ray's pixel, REF run_history :162-164): one
// Philox block when both lie in the same block, two otherwise.
__device__ __forceinline__ void rng_pair_at(const SlotRng& r, uint32_t j, uint32_t k0, uint32_t k1, uint32_t angle,
                                            double& u0, double& u1)
{
    const uint32_t m0 = (4u - r.pos) >> 1; // draws left in the buffered block
    uint32_t w[4];                         // the block holding draw j (its words)
    uint32_t q;                            // j's word offset in it (0 or 2)
    if (j < m0) {
        w[0] = r.b0, w[1] = r.b1, w[2] = r.b2, w[3] = r.b3;
        q = r.pos + 2 * j;
    } else {
        const uint32_t k = j - m0;
        philox_block(r.block + (k >> 1), r.photon, r.bin, angle, k0, k1, w[0], w[1], w[2], w[3]);
        q = (k & 1) ? 2u : 0u;
    }
    u0 = q == 0 ? words_to_uniform(w[0], w[1]) : words_to_uniform(w[2], w[3]);
    if (q == 0) { // j + 1 is the block's second draw
        u1 = words_to_uniform(w[2], w[3]);
        return;
    }
    u1 = rng_uniform_at(r, j + 1, k0, k1, angle); // j + 1 starts the next block
}

// Advance the stream past n draws (the state slot_uniform would leave).
__device__ __forceinline__ void rng_skip(SlotRng& r, uint32_t n, uint32_t k0, uint32_t k1, uint32_t angle)
{
    const uint32_t m0 = (4u - r.pos) >> 1;
    if (n <= m0) {
        r.pos += 2 * n;
        return;
    }
    const uint32_t rem = n - m0, nb = (rem + 1) >> 1;
    philox_block(r.block + nb - 1, r.photon, r.bin, angle, k0, k1, r.b0, r.b1, r.b2, r.b3);
    r.block += nb;
    r.pos = (rem & 1) ? 2 : 4;
}

// ----------------------------------------------------------------- mu table
// Linear attenuation lookup for the current ray's energy.  REG: <= 4 palette
// entries held in registers (4- or 8-bit palette); otherwise a per-lane table in
// shared memory: palette entries (P4) or mass attenuation per material
// (P8 / raw, multiplied by the voxel density at lookup).  Values are the
// products REF MuField forms (trace.cpp:10-20).
// Log-log evaluation of several tables at one energy.  When every material's
// mu table has the same energy knots (true for the reference's bundled data,
// checked at upload) the knot search and log(e) are shared; the arithmetic
// is that of tab_loglog (REF table.hpp:57-69), so values are identical.
// When the knots differ (e.g. a material with an absorption edge), each table
// gets its own knot search but log(e) is still computed once.
struct SharedLog {
    int i;
    bool exact, ok, has_le;
    double le;
    __device__ __forceinline__ void init(const TransportParams& P, double e, DevStatus* st, int bin,
                                         bool enabled = true)
    {
        ok = false;
        has_le = false;
        if (!P.shared_mu_grid || !enabled)
            return;
        const Tab t = mtab(P, P.mats[P.grid_mat].mu);
        if (!tab_locate(t, e, i, exact)) {
            raise(st, XS_E_OUT_OF_RANGE, kErrTableRange, bin, e, 0.0);
            return;
        }
        le = exact ? 0.0 : nl_log(e);
        has_le = !exact;
        ok = true;
    }
    __device__ __forceinline__ double eval(const TransportParams& P, TabDesc d, double e, DevStatus* st,
                                           int bin)
    {
        if (!ok) { // tab_loglog (REF table.hpp:57-69) with the shared log(e)
            const Tab t = mtab(P, d);
            int j;
            bool ex;
            if (!tab_locate(t, e, j, ex)) {
                raise(st, XS_E_OUT_OF_RANGE, kErrTableRange, bin, e, 0.0);
                return 0.0;
            }
            if (ex)
                return __ldg(t.y + j);
            const double y0 = __ldg(t.y + j), y1 = __ldg(t.y + j + 1);
            if (y0 <= 0.0 || y1 <= 0.0) {
                const double x0 = __ldg(t.x + j), x1 = __ldg(t.x + j + 1);
                const double u = (e - x0) / (x1 - x0);
                return y0 + u * (y1 - y0);
            }
            if (!has_le) {
                le = nl_log(e);
                has_le = true;
            }
            const double lx0 = __ldg(t.lx + j), lx1 = __ldg(t.lx + j + 1);
            const double u = (le - lx0) / (lx1 - lx0);
            return nl_exp(__ldg(t.ly + j) + u * (__ldg(t.ly + j + 1) - __ldg(t.ly + j)));
        }
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

// SM (walk kernel only): the <= 4 palette entries of REG in shared memory
// (T[c * kBlock]) instead of registers, for walk occupancy.
template <int FMT, bool REG, bool SM = false>
struct MuTab {
    double t0, t1, t2, t3;
    double* T;
    double energy;

    __device__ __noinline__ void fill(const TransportParams& P, double e, DevStatus* st, int bin)
    {
        fill_impl(P, e, st, bin);
    }
    __device__ __forceinline__ void fill_impl(const TransportParams& P, double e, DevStatus* st, int bin)
    {
        energy = e;
        if (REG) { // <= 4 palette entries in registers; one table evaluation per entry
            double v0 = 0.0, v1 = 0.0, v2 = 0.0, v3_ = 0.0;
            SharedLog sl;
            sl.init(P, e, st, bin);
            for (int c = 0; c < P.n_pal; ++c) {
                const int m = P.pal_mat[c];
                double mu = 0.0;
                if (m >= 1 && m < P.n_mats && P.mats[m].has_tables)
                    mu = sl.eval(P, P.mats[m].mu, e, st, bin) * (double)P.pal_dens[c];
                if (c == 0)
                    v0 = mu;
                else if (c == 1)
                    v1 = mu;
                else if (c == 2)
                    v2 = mu;
                else
                    v3_ = mu;
            }
            t0 = v0;
            t1 = v1;
            t2 = v2;
            t3 = v3_;
        } else if (FMT == kFmtP4) { // per palette entry
            for (int c = 0; c < P.n_pal; ++c)
                T[c * kBlock] = 0.0;
            SharedLog sl;
            sl.init(P, e, st, bin);
            for (int m = 1; m < P.n_mats; ++m) {
                const MatDesc& md = P.mats[m];
                const double ma = md.has_tables ? sl.eval(P, md.mu, e, st, bin) : 0.0;
                for (int c = 0; c < P.n_pal; ++c)
                    if (P.pal_mat[c] == m)
                        T[c * kBlock] = ma * (double)P.pal_dens[c];
            }
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
        if (REG && SM)
            return T[(code & 3) * kBlock];
        if (REG) {
            const double lo = (code & 1) ? t1 : t0;
            const double hi = (code & 1) ? t3 : t2;
            return (code & 2) ? hi : lo;
        }
        if (FMT == kFmtP4)
            return T[code * kBlock];
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
    uint32_t ucells;      // ... of which crossed a uniform cell / brick
};



template <int FMT, bool FAST>
__device__ __forceinline__ bool walk_begin_impl(const TransportParams& P, Walk& w, V3 o, V3 d,
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
    w.ucells = 0;
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
        // 1 / direction for the block march (walk_step); 0 for axes that do not move
        w.rdx = d.x != 0.0 ? 1.0 / d.x : 0.0;
        w.rdy = d.y != 0.0 ? 1.0 / d.y : 0.0;
        w.rdz = d.z != 0.0 ? 1.0 / d.z : 0.0;
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
    // 1/dt for the block walk's crossing counts (cross_n); axes that do not
    // move get the sentinel of start_axis<true>
    w.rdx = d.x != 0.0 ? fabs(d.x) * G.ihx : 1e-300;
    w.rdy = d.y != 0.0 ? fabs(d.y) * G.ihy : 1e-300;
    w.rdz = d.z != 0.0 ? fabs(d.z) * G.ihz : 1e-300;
    return true;
}

// Out-of-line copy (the megakernel keeps its instruction footprint small);
// the wavefront set-up kernel inlines walk_begin_impl so the walker state
// stays in registers instead of a local-memory frame.
template <int FMT, bool FAST>
__device__ __noinline__ bool walk_begin(const TransportParams& P, Walk& w, V3 o, V3 d, double target, bool march,
                                        DevStatus* st, int bin)
{
    return walk_begin_impl<FMT, FAST>(P, w, o, d, target, march, st, bin);
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

// Boundaries of one axis crossed by a step that ends at tm.  e = tn + k dt
// is the axis' last boundary inside the current block (k = boundaries left
// in it, 0 outside uniform blocks).  An axis whose block face is the step's
// exit (e <= tm, i.e. e == tm) crosses all k + 1; any other axis crosses the
// boundaries at or before tm, counted as trunc((tm - tn) / dt + 1) with the
// fp64 reciprocal (rd = |d| / h) and clamped to [0, k].  The count can be off
// by one only for a boundary within rounding of tm, which moves the depth by
// rounding-level amounts: the block walk already differs from REF at that
// level.  Outside uniform blocks (k = 0) this is exactly REF's step: the
// axes with tn == tm cross (trace.cpp:146-153).  Axes that do not move carry
// finite sentinels (tn = dt = 1e300, rd = 1e-300; start_axis<true>) so the
// estimate is 0 and tn + 0 * dt stays tn.
#ifndef XS_WALK_FMA
#define XS_WALK_FMA 1
#endif
// t-plane arithmetic of the block step, fused: tn + k dt with k = 0 or 1 is
// the same single rounding as REF's tn + dt, so voxel steps stay exact
__device__ __forceinline__ double plane_at(double tn, uint32_t k, double dt)
{
#if XS_WALK_FMA
    return __fma_rn(u2d_small(k), dt, tn);
#else
    return tn + u2d_small(k) * dt;
#endif
}
__device__ __forceinline__ int cross_n(double tn, double e, double rd, double tm, int k)
{
    // 2^52 + 1 + q rounded toward zero: its low word is trunc(q + 1) for q >= -1,
    // and negative (0xFFFFFFFx) just below, which the clamp turns into 0
    // (the count matters only for k > 0, inside blocks)
#if XS_WALK_FMA
    const int est = __double2loint(__fma_rz(tm - tn, rd, 4503599627370497.0));
#else
    const int est = __double2loint(__dadd_rz((tm - tn) * rd, 4503599627370497.0));
#endif
    const int n = est < 0 ? 0 : (est > k ? k : est);
    return e <= tm ? k + 1 : n;
}

// One voxel (REF trace.cpp:136-155 / :202-228).  Branch-free axis advance;
// the next voxel's load is issued before this step's fp64 chain and decoded
// only in the next step.
// RUN: the run field (Grid::run_*) is used along x (1), y (2), the axis the
// grid says (3, runtime), or not at all (0).
template <int FMT, bool REG, bool SKIP, int RUN = 3, bool SM = false>
__device__ __forceinline__ bool walk_step(const TransportParams& P, const MuTab<FMT, REG, SM>& tab,
                                          Walk& w)
{
    const Grid& G = P.G;
    if (w.march) { // REF trace.cpp:124-133
        const double ta = w.t + w.ix * w.dtx;
        const double tb = w.texit < ta + w.dtx ? w.texit : ta + w.dtx;
        const double tm = 0.5 * (ta + tb);
        const double px = w.ox + w.rx * tm, py = w.oy + w.ry * tm, pz = w.oz + w.rz * tm;
        const int vx = voxel_of(px, G.ox, G.ihx, G.nx), vy = voxel_of(py, G.oy, G.ihy, G.ny),
                  vz = voxel_of(pz, G.oz, G.ihz, G.nz);
        int code;
        float dens = 0.f;
        fetch<FMT>(G, vx, vy, vz, code, dens);
        const double mu = tab.mu(P, code & ~G.ubit, dens);
        if (SKIP) {
            // Block march: every later sample whose midpoint still lies in this
            // sample's uniform block (level bits) has the same mu, so their
            // segments are summed in one step (rounding-level change, like the
            // block walk).  Only for blocks that hold several samples.
            const int um = (1 << ((G.lvl_log2 >> (((uint32_t)code >> G.lvl_shift) << 2)) & 0xFu)) - 1;
            if (um + 1 >= 2 * P.step_voxels) {
                // the block's exit along the ray: the face ahead on each moving axis
                const double fx = G.ox + (double)(w.rx > 0.0 ? (vx | um) + 1 : (vx & ~um)) * G.hx;
                const double fy = G.oy + (double)(w.ry > 0.0 ? (vy | um) + 1 : (vy & ~um)) * G.hy;
                const double fz = G.oz + (double)(w.rz > 0.0 ? (vz | um) + 1 : (vz & ~um)) * G.hz;
                double tblk = w.rdx != 0.0 ? (fx - w.ox) * w.rdx : CUDART_INF;
                const double tyb = w.rdy != 0.0 ? (fy - w.oy) * w.rdy : CUDART_INF;
                const double tzb = w.rdz != 0.0 ? (fz - w.oz) * w.rdz : CUDART_INF;
                tblk = tyb < tblk ? tyb : tblk;
                tblk = tzb < tblk ? tzb : tblk;
                // the last sample j with midpoint t0 + (j + 1/2) h before the exit
                int j2 = (int)floor((tblk - w.t) * P.march_ih - 0.5);
                j2 = j2 > w.iy - 1 ? w.iy - 1 : j2;
                if (j2 > w.ix) {
                    const double te = w.t + (j2 + 1) * w.dtx;
                    w.depth += mu * ((w.texit < te ? w.texit : te) - ta);
                    w.skipped += (uint32_t)(j2 - w.ix);
                    ++w.ucells;
                    w.ix = j2 + 1;
                    return w.ix < w.iy;
                }
            }
        }
        w.depth += mu * (tb - ta);
        return ++w.ix < w.iy;
    }
    const int code = decode<FMT>(w.raw, w.shift);
    if (SKIP) {
        // One step = up to the next boundary crossing, or, in an aligned
        // uniform block (level field of the code), up to its exit: k* boundaries
        // of each axis remain inside the block (0 outside uniform blocks, where
        // this is exactly REF's voxel step).  Branch-free, so lanes in
        // uniform and mixed cells do not diverge.
        const int c = code & ~G.ubit;
        const int um = (1 << ((G.lvl_log2 >> (((uint32_t)code >> G.lvl_shift) << 2)) & 0xFu)) - 1;
        int kx = (w.sx > 0 ? ~w.ix : w.ix) & um;
        int ky = (w.sy > 0 ? ~w.iy : w.iy) & um;
        int kz = (w.sz > 0 ? ~w.iz : w.iz) & um;
        // the block's exit face per axis (k = 0: the next boundary, tn itself)
        double ex = plane_at(w.tnx, kx, w.dtx);
        double ey = plane_at(w.tny, ky, w.dty);
        double ez = plane_at(w.tnz, kz, w.dtz);
        double tm = ex;
        if (ey < tm)
            tm = ey;
        if (ez < tm)
            tm = ez;
        if (w.texit < tm)
            tm = w.texit;
        bool multi = um != 0;
        if (RUN != 0) {
            // The run ahead (Grid::run_*): a 1-voxel-wide box of r + 1 voxels
            // along the run axis, when the ray moves in the run's direction.
            // Taken instead of the block when the ray leaves it later (either
            // box is exact; picking by a cheaper rule, e.g. more boundaries
            // along the axis, measured no fewer steps on C3).
            const bool ax = RUN == 1 ? true : RUN == 2 ? false : G.run_axis == 0;
            int r = ((uint32_t)code >> G.run_shift) & G.run_mask;
            r = (ax ? w.sx : w.sy) == G.run_sign ? r : 0;
            const double ra = plane_at(ax ? w.tnx : w.tny, r, ax ? w.dtx : w.dty);
            const double ro = ax ? w.tny : w.tnx;
            double tr = ra < ro ? ra : ro;
            if (w.tnz < tr)
                tr = w.tnz;
            if (w.texit < tr)
                tr = w.texit;
            if (tr > tm) {
                tm = tr;
                kx = ax ? r : 0;
                ky = ax ? 0 : r;
                kz = 0;
                ex = ax ? ra : ro;
                ey = ax ? ro : ra;
                ez = w.tnz;
                multi = true;
            }
        }
        const double mu = tab.mu(P, c, w.dens);
        const double seg = mu * (tm - w.t);
        const double nd = w.depth + seg;
        if (nd >= w.target) { // free path ends in this voxel / block; t_hit in hit_t()
            w.hit = 1;
            w.mu_hit = mu;
            w.texit = tm;
            return false;
        }
        const int nx = cross_n(w.tnx, ex, w.rdx, tm, kx);
        const int ny = cross_n(w.tny, ey, w.rdy, tm, ky);
        const int nz = cross_n(w.tnz, ez, w.rdz, tm, kz);
        const int nix = w.ix + nx * w.sx, niy = w.iy + ny * w.sy, niz = w.iz + nz * w.sz;
        const bool inside = (tm < w.texit) && (uint32_t)nix < (uint32_t)G.nx &&
                            (uint32_t)niy < (uint32_t)G.ny && (uint32_t)niz < (uint32_t)G.nz;
        // (an axis that does not cross keeps its term: term_x(nix) == ax)
        const uint32_t nax = term_x(G, nix), nay = term_y(G, niy), naz = term_z(G, niz);
        if (inside)
            prefetch<FMT>(G, nax + nay + naz, w.raw, w.shift, w.dens);
        w.depth = nd;
        w.t = tm;
        // (n = 0: tn + 0 * dt == tn, dt finite)
        w.tnx = plane_at(w.tnx, nx, w.dtx);
        w.tny = plane_at(w.tny, ny, w.dty);
        w.tnz = plane_at(w.tnz, nz, w.dtz);
        if (multi) {
            w.skipped += (uint32_t)(nx + ny + nz) - 1u;
            ++w.ucells;
        }
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

// A history's total into its bin's Sum t and Sum t^2 (REF run_history :225-228).
__device__ __forceinline__ void bin_total_add(const TransportParams& P, const Block& B, int bin, double t,
                                              DevStatus* st)
{
    if (t != 0.0) {
        unsigned long long* bs = B.bins + 8 * bin;
        if (!tally_limbs(bs, t, P.log2_img) || !tally_limbs(bs + 3, t * t, 2 * P.log2_img))
            raise(st, XS_E_RUNTIME, kErrTallyOverflow, bin, 0.0, t);
    }
}

// History end (REF run_history :225-241): bin statistics from the exact
// fixed-point history total, per-pixel grouping for the variance, free slot.
// release = false: the caller frees the slot itself.
template <class Q>
__device__ __noinline__ void finalize_history(const TransportParams& P, const Block& B, const Q qs, int s,
                                              uint64_t var_base, DevStatus* st, bool release = true)
{
    Slot& S = qs.slot(s);
    const double t = dequantize(S.T[0], S.T[1], S.T[2], P.log2_img);
    qs.bin_total(P, B, S.bin, t, st);
    if (P.track_var) {
        const uint32_t* vp = P.var_pix + var_base;
        const double* vv = P.var_val + var_base;
        const int n = S.n_var < P.var_cap ? S.n_var : P.var_cap;
        for (int a = 0; a < n; ++a) {
            const uint32_t pa = vp[a];
            if (pa >= (uint32_t)P.nu * (uint32_t)P.nv) { // corrupt scratch: report, never write out of bounds
                raise(st, XS_E_RUNTIME, kErrStuck, S.bin, S.E, 14.0);
                continue;
            }
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
    qs.history_done(B);
    if (release)
        qs.release(s);
}

template <class Q>
__device__ __forceinline__ void end_history(const TransportParams& P, const Block& B, const Q qs, int s,
                                            uint64_t var_base, DevStatus* st)
{
    qs.fence(); // this lane's tallies / scratch before the hand-off
    if (atomicSub(&qs.slot(s).pending, 1) == 1)
        finalize_history(P, B, qs, s, var_base, st);
}

// Scoring-ray completion (REF run_history :178-193): the point-detector
// score tpre * exp(-tau) into the pixel's limbs and the history total, the
// variance scratch, and the ray's share of the history's pending count.
template <class Q>
__device__ __forceinline__ void score_complete(const TransportParams& P, const Block& B, const Q& qs, int s,
                                               uint32_t pix, double tpre, double depth, uint64_t var_base,
                                               DevStatus* st)
{
    Slot& S = qs.slot(s);
    const double x = tpre * nl_exp(-depth);
    uint64_t l0 = 0, l1 = 0, l2 = 0;
    if (!isfinite(x)) {
        raise(st, XS_E_RUNTIME, kErrNonFinite, S.bin, S.e_in, x);
    } else if (!quantize(ldexp(x, -P.log2_img), l0, l1, l2)) {
        raise(st, XS_E_RUNTIME, kErrTallyOverflow, S.bin, S.e_in, x);
    } else {
        unsigned long long* img = P.accum + P.off_image + 4ull * pix;
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
            P.var_pix[var_base + k] = pix;
            P.var_val[var_base + k] = x;
        }
    }
    end_history(P, B, qs, s, var_base, st);
}

// REF run_history :162-164: the scoring pixel of one (u, v) draw pair.
__device__ __forceinline__ uint32_t score_pixel(const TransportParams& P, double uu, double uv)
{
    int iu = (int)(uu * P.nu);
    int iv = (int)(uv * P.nv);
    iu = iu < P.nu - 1 ? iu : P.nu - 1;
    iv = iv < P.nv - 1 ? iv : P.nv - 1;
    return (uint32_t)(iv * P.nu + iu);
}

// Free-path completion: the reference's per-history event logic
// (run_history :141-223) on the history's own Philox stream, in two phases:
// event_select (escape / interaction choice / the scoring rays, REF
// :141-194) returns the interaction kind, and event_continue (the scattered
// photon, cap and roulette, REF :195-223) follows for Compton and Rayleigh.
// The stream is handed over in the slot, so the wavefront engine can run the
// two phases for different lanes (continuations gathered by kind).
template <int FMT, class Q>
__device__ __noinline__ int event_select(const TransportParams& P, const Block& B, const Q qs, int s,
                                         bool hit, double t_hit, int vix, int viy, int viz,
                                         uint64_t var_base, DevStatus* st)
{
    Slot& S = qs.slot(s);
    const int bin = S.bin;
    const double W = S.W;
    if (!hit) {
        qs.ledger(P, B, 1, W, st, bin);
        end_history(P, B, qs, s, var_base, st);
        return K_NONE;
    }
    SlotRng rng = S.rng;
    const V3 dir = v3(S.dx, S.dy, S.dz);
    const V3 pos = v3(S.px, S.py, S.pz) + dir * t_hit;
    int code;
    float dens;
    fetch<FMT>(P.G, vix, viy, viz, code, dens);
    const int mat = material_of<FMT>(P, code & ~P.G.ubit);
    if (mat <= 0 || mat >= P.n_mats) { // an interaction needs matter: corrupt state
        raise(st, XS_E_RUNTIME, kErrStuck, bin, S.E, 15.0);
        end_history(P, B, qs, s, var_base, st);
        return K_NONE;
    }
    const MatDesc& md = P.mats[mat];
    const double E = S.E;
    // select_interaction (cross_sections.cpp:81-96); one knot search and one
    // log(E) for the three tables when they share the energy knots
    SharedLog sl;
    sl.init(P, E, st, bin, P.shared_e_grid != 0);
    const double pe = sl.eval(P, md.pe, E, st, bin);
    const double incoh = sl.eval(P, md.incoh, E, st, bin);
    const double coh = sl.eval(P, md.coh, E, st, bin);
    const double total = pe + incoh + coh;
    if (!(total > 0.0))
        raise(st, XS_E_RUNTIME, kErrSigmaAll, bin, E, (double)mat);
    const double u = slot_uniform(&rng, P.k0, P.k1, P.angle) * total;
    const int kind = u < pe ? K_PE : (u < pe + incoh ? K_COMPTON : K_RAYLEIGH);
    if (kind == K_PE) {
        qs.ledger(P, B, 2, W, st, bin);
        end_history(P, B, qs, s, var_base, st);
        return K_PE;
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
    if constexpr (Q::kBatchScores) {
        // one batch entry; the set-up kernel draws its pixels in parallel
        qs.push_score_batch(s, rng, kind);
        rng_skip(rng, 2u * (uint32_t)P.splitting, P.k0, P.k1, P.angle);
    } else {
        const uint32_t qbase = qs.reserve_scores(P.splitting);
#pragma unroll 1
        for (int k = 0; k < P.splitting; ++k) { // REF :162-164 pixel draws
            const double uu = slot_uniform(&rng, P.k0, P.k1, P.angle); // u first, then v
            const double uv = slot_uniform(&rng, P.k0, P.k1, P.angle);
            qs.push_score(qbase + k, s, score_pixel(P, uu, uv));
        }
    }
    S.rng = rng;
    return kind;
}

template <class Q>
__device__ __noinline__ void event_continue(const TransportParams& P, const Block& B, const Q qs, int s,
                                            uint64_t var_base, DevStatus* st)
{
    Slot& S = qs.slot(s);
    SlotRng rng = S.rng;
    const int bin = S.bin;
    const double W = S.W;
    const double E = S.e_in;
    const int kind = S.kind;
    const V3 dir = v3(S.ix, S.iy, S.iz);
    const MatDesc& md = P.mats[S.mat];
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
            // trials are bounded (2^24 draws) so corrupt state raises instead of hanging
            uint32_t trials = 0;
            for (;;) {
                if (trials > (1u << 24)) {
                    raise(st, XS_E_RUNTIME, kErrStuck, bin, E, 1.0 + S.mat);
                    break;
                }
                const double t = 1.0 + 2.0 * alpha; // kahn_sample_cos_theta, samplers.cpp:12-30
                double cos_th = 1.0;
                for (;; ++trials) {
                    if (trials > (1u << 24))
                        break;
                    const double r1 = slot_uniform(&rng, P.k0, P.k1, P.angle);
                    const double r2 = slot_uniform(&rng, P.k0, P.k1, P.angle);
                    const double r3 = slot_uniform(&rng, P.k0, P.k1, P.angle);
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
                if (slot_uniform(&rng, P.k0, P.k1, P.angle) * s_max <= sv) {
                    ap = alpha / (1.0 + alpha * (1.0 - nl_cos(theta)));
                    phi = 2.0 * kPi * slot_uniform(&rng, P.k0, P.k1, P.angle);
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
            for (uint32_t trials = 0;; ++trials) {
                if (trials > (1u << 24)) {
                    raise(st, XS_E_RUNTIME, kErrStuck, bin, E, 200.0 + S.mat);
                    break;
                }
                const double qq = invert_mass(P, md, slot_uniform(&rng, P.k0, P.k1, P.angle) * tot, q_max);
                const double sh = 1.0 < qq * scale ? 1.0 : qq * scale;
                const double cos_th = 1.0 - 2.0 * sh * sh;
                if (slot_uniform(&rng, P.k0, P.k1, P.angle) * 2.0 <= 1.0 + cos_th * cos_th) {
                    const double cc = cos_th < -1.0 ? -1.0 : (1.0 < cos_th ? 1.0 : cos_th);
                    theta = nl_acos(cc);
                    phi = 2.0 * kPi * slot_uniform(&rng, P.k0, P.k1, P.angle);
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
        qs.ledger(P, B, 3, W, st, bin);
        alive = false;
    } else if (S.wmin > 0.0 && W < S.wmin) { // REF :213-222
        if (slot_uniform(&rng, P.k0, P.k1, P.angle) < P.survival) {
            const double boosted = W / P.survival;
            qs.ledger(P, B, 5, boosted - W, st, bin);
            Wn = boosted;
        } else {
            qs.ledger(P, B, 4, W, st, bin);
            alive = false;
        }
    }
    if (alive) {
        S.W = Wn;
        S.target = -nl_log(slot_uniform(&rng, P.k0, P.k1, P.angle));
        S.rng = rng;
        qs.push_free(s);
    } else {
        end_history(P, B, qs, s, var_base, st);
    }
}

template <int FMT, class Q>
__device__ __forceinline__ void history_event(const TransportParams& P, const Block& B, const Q qs, int s,
                                              bool hit, double t_hit, int vix, int viy, int viz,
                                              uint64_t var_base, DevStatus* st)
{
    const int kind = event_select<FMT>(P, B, qs, s, hit, t_hit, vix, viy, viz, var_base, st);
    if (kind == K_COMPTON || kind == K_RAYLEIGH)
        event_continue(P, B, qs, s, var_base, st);
}

// History start (REF run_history :120-138, sample_emission :73-87).
// Returns the history's initial weight w0; tally_w0 = false leaves its ledger
// entry ("initial") to the caller (the wavefront admission sums it in
// registers instead of contended shared-memory atomics).
template <class Q>
__device__ __noinline__ double history_start(const TransportParams& P, const Block& B, const Q qs,
                                             const uint64_t* sstart, int s, uint64_t h, DevStatus* st,
                                             bool tally_w0 = true)
{
    Slot& S = qs.slot(s);
    int lo = 0, hi = P.n_bins; // last bin b with start[b] <= h (skips empty bins)
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (sstart[mid] <= h)
            lo = mid;
        else
            hi = mid;
    }
    const int bin = lo;
    SlotRng rng;
    rng.photon = (uint32_t)(h - sstart[lo]);
    rng.bin = (uint32_t)lo;
    rng.block = 0;
    rng.pos = 4;
    const double u1 = slot_uniform(&rng, P.k0, P.k1, P.angle);
    const double u2 = slot_uniform(&rng, P.k0, P.k1, P.angle);
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
    const double E = __ldg(P.bin_energy + bin);
    if (tally_w0)
        ledger_add(P, B, 0, w0, st, bin);
    const double target_mfp = -nl_log(slot_uniform(&rng, P.k0, P.k1, P.angle));
    if constexpr (Q::kBatchScores) {
        // global slot (wavefront engine): the fields this writes, as 16-byte
        // stores (a warp's scattered slots cost one L1 wavefront per lane per
        // store instruction; the interaction record ix..pref is left alone)
        double2* q = reinterpret_cast<double2*>(&S);
        q[0] = make_double2(src.x, src.y);
        q[1] = make_double2(src.z, dir.x);
        q[2] = make_double2(dir.y, dir.z);
        q[3] = make_double2(E, w0);
        q[4] = make_double2(P.wmin_rel * w0, target_mfp);
        uint4* u = reinterpret_cast<uint4*>(&S.T[0]);
        u[0] = make_uint4(0u, 0u, 0u, 0u);                                   // T[0], T[1]
        u[1] = make_uint4(0u, 0u, rng.photon, rng.bin);                       // T[2], rng
        u[2] = make_uint4(rng.block, rng.pos, rng.b0, rng.b1);
        u[3] = make_uint4(rng.b2, rng.b3, (uint32_t)bin, 0u);                 // ..., bin, gen
        u[4] = make_uint4(0u, 0u, 1u, 0u); // kind, mat (set by the interaction), pending, n_var
    } else {
        S.px = src.x;
        S.py = src.y;
        S.pz = src.z;
        S.dx = dir.x;
        S.dy = dir.y;
        S.dz = dir.z;
        S.E = E;
        S.W = w0;
        S.wmin = P.wmin_rel * w0;
        S.T[0] = S.T[1] = S.T[2] = 0ull;
        S.bin = bin;
        S.gen = 0;
        S.pending = 1;
        S.n_var = 0;
        S.target = target_mfp;
        S.rng = rng;
    }
    qs.push_free(s);
    qs.claim(s);
    return w0;
}

// Scoring-ray set-up (REF run_history :166-183): geometry, p(theta), e_out,
// response; returns the score prefactor (point_detector_score without exp(-tau)).
__device__ __forceinline__ double score_setup(const TransportParams& P, const Slot& S, uint32_t pix,
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

} // namespace xsd
