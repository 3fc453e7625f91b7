// wavefront.cu — the scatter transport as a pipeline of small kernels
// (REF transport.cpp:114-324, same per-history arithmetic as transport.cu).
//
// The megakernel (transport.cu) runs set-up, walking and event logic in one
// persistent kernel.  On B200 it is bound by instruction-cache misses: about
// 40 KB of set-up code per ray against a 32 KB L1.5 I-cache.  It also idles
// half its lanes, because a warp walks 32 rays until the longest ends
// (profiles/r1_bench_kernel_ncu.md).  Here every stage is its own kernel over
// a global queue, so each kernel's code stays resident and its warps are
// coherent:
//
//   setup    one thread per queued task: scoring geometry + p(theta) + e_out
//            (REF :166-183) or the free path's start; mu table; Siddon init.
//            Writes a compact walker state (SoA, coalesced).
//   walk     persistent; a lane that finishes a ray takes the next state from
//            the queue (refills batched per warp), so lanes stay busy.  Only
//            the Siddon loop is resident.
//   complete one thread per finished ray: scoring tally (REF :178-193) or the
//            history's event (REF :141-223), which pushes the next wave's
//            scoring rays and free path.
//   plan     one thread: admit new histories into released slots.
//   admit    one thread per admitted history (REF :120-138).
//
// Per wave, each live history advances by one free path.  The scoring rays of
// its last interaction ride in the same wave.  A history's slot is only
// rewritten by `complete`, after `setup` has copied everything the wave's
// rays need, so the interaction record needs no double buffering.  Tallies
// are the same fixed-point integers as the megakernel's, so both engines give
// bit-identical images and statistics.

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <unistd.h>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "capi_internal.h"
#include "transport_core.cuh"

namespace xsd {

// Data-driven indices are validated before use: a violation (which would
// mean corrupt pipeline state) raises a device error naming the site instead
// of touching memory out of bounds.
#define XS_GUARD(cond, st, site) (__builtin_expect(!!(cond), 1) ? true : (raise((st), XS_E_RUNTIME, kErrStuck, 0, 0.0, (site)), false))

namespace {

#ifndef XSW_REFILL_EXACT
#define XSW_REFILL_EXACT 4 // the voxel walk refills sooner (its steps are short): -3%
#endif
#ifndef XSW_EXACT_BLOCKS
#define XSW_EXACT_BLOCKS 7 // the voxel walk: 72 registers
#endif
#ifndef XSW_REFILL
#define XSW_REFILL 8
#endif
// minimum resident blocks per SM of the latency-bound kernels: register caps
// that trade a few spills for occupancy (XSCAT_KTIME, C3, one pipeline, same
// box: set-up 84.6 -> 72.5 ms at 64 registers, scoring 26.6 -> 22.0 ms at 40,
// events 60.0 -> 53.0 ms at 80; admission is faster uncapped; later, with the
// walk at seven blocks: set-up 67.1 -> 65.8 ms at 72 registers, events and
// scoring unchanged at 5 / 7 and 10 / 16 blocks)
#ifndef XSW_SETUP_MINB
#define XSW_SETUP_MINB 7
#endif
#ifndef XSW_SCORE_MINB
#define XSW_SCORE_MINB 12
#endif
#ifndef XSW_EVENT_MINB
#define XSW_EVENT_MINB 6
#endif
#ifndef XSW_ADMIT_MINB
#define XSW_ADMIT_MINB 1
#endif
#ifndef XSW_WALK_MU_SMEM
#define XSW_WALK_MU_SMEM 1 // walk: the register mu table (<= 4 palette entries) in shared memory
#endif
#ifndef XSW_INNER
#define XSW_INNER 3 // block steps per walk-loop trip between the warp's refill checks
                    // (C3 walk: 1 -> 212, 2 -> 200, 3 -> 193, 4 -> 204, 5 -> 201 ms)
#endif
constexpr int kRefill = XSW_REFILL; // idle lanes that trigger a warp's refill in the walk kernel

#ifndef XSW_WALK_BLOCKS
#define XSW_WALK_BLOCKS 7 // resident block-walk blocks per SM (8-bit palette): 72 registers, no
                          // spills once the register mu table lives in shared memory (C3 walk
                          // 189 -> 178 ms; 8 blocks spill); the 4-bit and march walks keep 6
#endif

// A history's scoring rays of one interaction: the slot and its Philox
// stream at the first pixel draw (the set-up kernel draws pixel k from
// draws 2k, 2k+1, REF run_history :162-164).
struct ScoreBatch {
    uint32_t slot;
    SlotRng rng;
};

struct alignas(8) WaveQueue {
    ScoreBatch* batch; // one per interaction, splitting rays each: Compton from the
                       // front, Rayleigh from the back (batch[cap - 1 - k]), so set-up
                       // warps rarely mix the two kinds' branches
    uint32_t* free;    // slot
    uint32_t n_batch, n_batch_r; // (one 64-bit word: a warp reserves both ends in one atomic)
    uint32_t n_free, cap;
};

// batch b of a wave's scoring work (Compton batches first, then Rayleigh)
__device__ __forceinline__ const ScoreBatch& batch_at(const WaveQueue& q, uint32_t b)
{
    return b < q.n_batch ? q.batch[b] : q.batch[q.cap - 1u - (b - q.n_batch)];
}

struct WaveCtl {
    WaveQueue q[2];
    uint32_t* free_stack; // released slots, [0, free_top)
    int32_t free_top;
    uint32_t* fin;        // histories whose last scoring ray the wave's scoring kernel counted
    uint32_t n_fin;       //   down, finalized by the wave's event kernel (reset by set-up)
    uint32_t cursor;      // walk kernel work cursor
    uint32_t ev_cursor;   // event kernel work cursor
    uint32_t setup_cursor; // set-up kernel work cursor (reset by wave_plan)
    uint32_t n_rays, n_score;
    uint32_t admit_n, live;
    unsigned long long next_h, admit_base;
    uint32_t waves, admit_q;
};

// Walker state between the set-up and walk kernels (structure of arrays over
// the wave's rays, so a warp's loads and stores coalesce).
struct WaveRays {
    double *t, *texit, *target, *tn, *dt, *mu; // tn, dt: 3 planes; mu: n_mu planes
    double* rd;                                // 3 planes: 1/dt (block walk crossing counts)
    int* vox;                                  // 3 planes: ix, iy, iz
    uint8_t* flags;                            // (sx+1) | (sy+1) << 2 | (sz+1) << 4 | walking << 6
    double* pre;                               // scoring prefactor (set-up -> complete)
    uint32_t* pix;                             // scoring pixel (set-up -> complete)
    double* res;                               // depth (scoring) / t_hit (free path)
    int* res_vox;                              // 3 planes: the free path's interaction voxel
    uint8_t* res_hit;
    uint32_t cap;
    int32_t n_mu;
};

struct WaveArgs {
    Slot* slots;
    WaveCtl* ctl;
    WaveRays R;
    unsigned long long* next_h; // next history to admit, shared by the pipelines
    uint32_t n_slots;
    int32_t cur; // queue consumed by this wave (the other one is filled)
};

// Queue pushes of the event code, deferred to a point where the warp has
// reconverged.  The event functions run in deeply divergent code (rejection
// loops of different lengths, __noinline__ calls); warp-aggregated
// reservations there (__activemask + __shfl_sync) hung the event kernel on
// some inputs.  Each lane records at most one push of each kind per window
// and the kernel flushes them with full-warp ballots (flush_deferred).
struct Deferred {
    int32_t batch_slot, free_slot, rel_slot, batch_rayleigh;
    SlotRng rng;
};

// Queue policy of the wavefront engine (see transport_core.cuh).
struct GlobalQ {
    Slot* slots;
    WaveCtl* ctl;
    int out;
    int free_at;    // >= 0: this thread's free-path entry is pre-reserved (admission)
    Deferred* def;  // this lane's deferred pushes
    __device__ __forceinline__ Slot& slot(int s) const { return slots[s]; }
    static constexpr bool kBatchScores = true;
    __device__ __forceinline__ void push_score_batch(int s, const SlotRng& r, int kind) const
    {
        if (def->batch_slot < 0) {
            def->batch_slot = s;
            def->batch_rayleigh = kind == K_RAYLEIGH ? 1 : 0;
            def->rng = r;
            return;
        }
        WaveQueue& q = ctl->q[out]; // (a second push in one window: not aggregated)
        const uint32_t i = kind == K_RAYLEIGH ? q.cap - 1u - atomicAdd(&q.n_batch_r, 1u) : atomicAdd(&q.n_batch, 1u);
        q.batch[i].slot = (uint32_t)s;
        q.batch[i].rng = r;
    }
    // (per-ray pushes: megakernel only)
    __device__ __forceinline__ uint32_t reserve_scores(int) const { return 0; }
    __device__ __forceinline__ void push_score(uint32_t, int, uint32_t) const {}
    __device__ __forceinline__ void push_free(int s) const
    {
        WaveQueue& q = ctl->q[out];
        if (free_at >= 0)
            q.free[free_at] = (uint32_t)s;
        else if (def->free_slot < 0)
            def->free_slot = s;
        else
            q.free[atomicAdd(&q.n_free, 1u)] = (uint32_t)s;
    }
    __device__ __forceinline__ void claim(int) const {}
    __device__ __forceinline__ void release(int s) const
    {
        if (def->rel_slot < 0) {
            def->rel_slot = s;
            return;
        }
        ctl->free_stack[atomicAdd(&ctl->free_top, 1)] = (uint32_t)s;
    }
    // (end_history's hand-off: in the wavefront engine only the event kernel
    // ends histories through it, one event per history per launch, and the
    // finalizer of a history it does not end runs in a later launch; kernel
    // boundaries order the writes, so no fence is needed)
    __device__ __forceinline__ void fence() const {}
    // statistics straight into the block's shared accumulators (folding them
    // per warp at the flush points, like the pushes, measured slower: event
    // kernel 58 -> 67 ms per C3 projection)
    __device__ __forceinline__ void ledger(const TransportParams& P, const Block& B, int k, double w,
                                           DevStatus* st, int bin) const
    {
        ledger_add(P, B, k, w, st, bin);
    }
    __device__ __forceinline__ void bin_total(const TransportParams& P, const Block& B, int bin, double t,
                                              DevStatus* st) const
    {
        bin_total_add(P, B, bin, t, st);
    }
    __device__ __forceinline__ void history_done(const Block& B) const { sadd(B.diag + 2, 1); }
};

__device__ __forceinline__ void deferred_reset(Deferred& d)
{
    d.batch_slot = d.free_slot = d.rel_slot = -1;
    d.batch_rayleigh = 0;
}

// All 32 lanes, converged: one reservation per queue for the warp's pushes.
__device__ __forceinline__ void flush_deferred(const TransportParams& P, const Block& B, WaveCtl* ctl, int out,
                                               Deferred& d, uint32_t n_slots, DevStatus* st)
{
    (void)P;
    (void)B;
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    WaveQueue& q = ctl->q[out];
    const unsigned mb = __ballot_sync(kFull, d.batch_slot >= 0);
    if (mb) { // Compton batches from the front, Rayleigh ones from the back
        const unsigned mr = __ballot_sync(kFull, d.batch_slot >= 0 && d.batch_rayleigh), mc = mb & ~mr;
        unsigned long long both = 0;
        if (lane == 0)
            both = atomicAdd(reinterpret_cast<unsigned long long*>(&q.n_batch),
                             (unsigned long long)__popc(mc) | ((unsigned long long)__popc(mr) << 32));
        both = __shfl_sync(kFull, both, 0);
        const uint32_t bc = (uint32_t)both, br = (uint32_t)(both >> 32);
        if (d.batch_slot >= 0) {
            const uint32_t k = d.batch_rayleigh ? br + (uint32_t)__popc(mr & lt) : bc + (uint32_t)__popc(mc & lt);
            if (XS_GUARD(k < n_slots, st, 16.0)) {
                const uint32_t i = d.batch_rayleigh ? q.cap - 1u - k : k;
                q.batch[i].slot = (uint32_t)d.batch_slot;
                q.batch[i].rng = d.rng;
            }
        }
    }
    const unsigned mf = __ballot_sync(kFull, d.free_slot >= 0);
    if (mf) {
        uint32_t base = 0;
        if (lane == 0)
            base = atomicAdd(&q.n_free, (uint32_t)__popc(mf));
        base = __shfl_sync(kFull, base, 0);
        if (d.free_slot >= 0) {
            if (XS_GUARD(base + (uint32_t)__popc(mf & lt) < n_slots, st, 17.0))
                q.free[base + (uint32_t)__popc(mf & lt)] = (uint32_t)d.free_slot;
        }
    }
    const unsigned mr = __ballot_sync(kFull, d.rel_slot >= 0);
    if (mr) {
        int32_t base = 0;
        if (lane == 0)
            base = atomicAdd(&ctl->free_top, (int32_t)__popc(mr));
        base = __shfl_sync(kFull, base, 0);
        if (d.rel_slot >= 0) {
            if (XS_GUARD((uint32_t)(base + __popc(mr & lt)) < n_slots, st, 18.0))
                ctl->free_stack[base + __popc(mr & lt)] = (uint32_t)d.rel_slot;
        }
    }
    deferred_reset(d);
}

__device__ __forceinline__ uint64_t var_base_of(const TransportParams& P, int s)
{
    return (uint64_t)s * (uint64_t)P.var_cap;
}

// Shared-memory statistics of a block (bins, ledger, diagnostics), flushed to
// the global accumulator when the block ends.
// Layout: bins (8 per bin), diag (8), then one 24-word ledger per warp: every
// history end adds to a ledger word, and 64-bit shared atomics are
// compare-and-swap loops, so per-warp copies keep the contention inside a warp.
constexpr int kStatWarps = kBlock / 32;
__host__ __device__ constexpr size_t stat_words(int n_bins) { return 8 * (size_t)n_bins + 8 + 24 * kStatWarps; }

__device__ __forceinline__ Block block_stats(const TransportParams& P, unsigned long long* smem)
{
    Block B;
    B.bins = smem;
    B.diag = B.bins + 8 * P.n_bins;
    B.ledger = B.diag + 8 + 24 * (threadIdx.x >> 5);
    for (int i = threadIdx.x; i < (int)stat_words(P.n_bins); i += blockDim.x)
        B.bins[i] = 0ull;
    __syncthreads();
    return B;
}

__device__ __forceinline__ void flush_stats(const TransportParams& P, const Block& B)
{
    __syncthreads();
    for (int i = threadIdx.x; i < 8 * P.n_bins; i += blockDim.x)
        if (B.bins[i])
            red_add(P.accum + P.off_bins + i, B.bins[i]);
    const unsigned long long* led = B.diag + 8; // every warp's ledger
    for (int i = threadIdx.x; i < 24; i += blockDim.x) {
        unsigned long long v = 0;
        for (int w = 0; w < kStatWarps; ++w)
            v += led[24 * w + i];
        if (v)
            red_add(P.accum + P.off_ledger + i, v);
    }
    for (int i = threadIdx.x; i < 8; i += blockDim.x)
        if (B.diag[i])
            red_add(P.accum + P.off_diag + i, B.diag[i]);
}

template <int FMT, bool REG>
__device__ __forceinline__ void store_mu(const WaveRays& R, uint32_t i, const MuTab<FMT, REG>& tab)
{
    if (REG) {
        __stcs(&R.mu[i], tab.t0);
        __stcs(&R.mu[R.cap + i], tab.t1);
        __stcs(&R.mu[2ull * R.cap + i], tab.t2);
        __stcs(&R.mu[3ull * R.cap + i], tab.t3);
    } else {
        for (int c = 0; c < R.n_mu; ++c)
            R.mu[(uint64_t)c * R.cap + i] = tab.T[c * kBlock];
    }
}

template <int FMT, bool REG, bool SM>
__device__ __forceinline__ void load_mu(const WaveRays& R, uint32_t i, MuTab<FMT, REG, SM>& tab)
{
    if (REG && SM) {
        for (int c = 0; c < 4; ++c)
            tab.T[c * kBlock] = __ldcs(&R.mu[(uint64_t)c * R.cap + i]);
    } else if (REG) {
        tab.t0 = __ldcs(&R.mu[i]);
        tab.t1 = __ldcs(&R.mu[R.cap + i]);
        tab.t2 = __ldcs(&R.mu[2ull * R.cap + i]);
        tab.t3 = __ldcs(&R.mu[3ull * R.cap + i]);
    } else {
        for (int c = 0; c < R.n_mu; ++c)
            tab.T[c * kBlock] = R.mu[(uint64_t)c * R.cap + i];
    }
}

// ------------------------------------------------------------------ set-up
// MARCH (step_voxels > 1, REF trace.cpp:116-134): scoring rays are midpoint
// marches; their walker state is the origin (tn planes), the direction (dt
// planes), t0, t1 and the sample count (vox plane 1), flagged 128.  Free paths
// are always exact Siddon walks (REF trace.cpp:189-230).
template <int FMT, bool REG, bool SKIP, bool MARCH>
__global__ void __launch_bounds__(kBlock, XSW_SETUP_MINB) wave_setup(const __grid_constant__ TransportParams P,
                                                     const __grid_constant__ WaveArgs A)
{
    extern __shared__ __align__(16) unsigned char smem[];
    WaveCtl* ctl = A.ctl;
    const WaveQueue& in = ctl->q[A.cur];
    const uint32_t n_s = (in.n_batch + in.n_batch_r) * (uint32_t)P.splitting, n = n_s + in.n_free;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        ctl->cursor = 0;
        ctl->ev_cursor = 0;
        ctl->n_rays = n;
        ctl->n_score = n_s;
        ctl->n_fin = 0;
        ctl->q[A.cur ^ 1].n_batch = 0;
        ctl->q[A.cur ^ 1].n_batch_r = 0;
        ctl->q[A.cur ^ 1].n_free = 0;
    }
    MuTab<FMT, REG> tab;
    tab.T = reinterpret_cast<double*>(smem) + threadIdx.x;
    tab.energy = -1.0;
    DevStatus* st = P.status;
    const WaveRays& R = A.R;
    uint32_t c_rays = 0;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        Walk w;
        w.march = 0;
        bool walking;
        if (i < n_s) { // REF run_history :162-183
            const uint32_t b = i / (uint32_t)P.splitting, k = i - b * (uint32_t)P.splitting;
            const ScoreBatch& sb = batch_at(in, b);
            const Slot& S = A.slots[sb.slot];
            double uu, uv;
            rng_pair_at(sb.rng, 2 * k, P.k0, P.k1, P.angle, uu, uv);
            const uint32_t pix = score_pixel(P, uu, uv);
            __stcs(&R.pix[i], pix);
            V3 o, to_det;
            double e_out;
            __stcs(&R.pre[i], score_setup(P, S, pix, o, to_det, e_out, st));
            if (tab.energy != e_out) // REF trace_attenuation builds MuField(e_out)
                tab.fill_impl(P, e_out, st, S.bin);
            walking = walk_begin_impl<FMT, SKIP>(P, w, o, to_det, CUDART_INF, MARCH, st, S.bin);
            ++c_rays;
        } else { // REF trace.cpp:189-230
            const Slot& S = A.slots[in.free[i - n_s]];
            if (tab.energy != S.E)
                tab.fill_impl(P, S.E, st, S.bin);
            walking = walk_begin_impl<FMT, SKIP>(P, w, v3(S.px, S.py, S.pz), v3(S.dx, S.dy, S.dz), S.target,
                                            false, st, S.bin);
        }
        if (!walking) { // misses the grid: zero depth, no interaction
            R.flags[i] = 0;
            R.res[i] = 0.0;
            R.res_hit[i] = 0;
            continue;
        }
        __stcs(&R.t[i], w.t);
        __stcs(&R.texit[i], w.texit);
        __stcs(&R.target[i], w.target);
        if (MARCH && w.march) {
            __stcs(&R.tn[i], w.ox);
            __stcs(&R.tn[R.cap + i], w.oy);
            __stcs(&R.tn[2ull * R.cap + i], w.oz);
            __stcs(&R.dt[i], w.rx);
            __stcs(&R.dt[R.cap + i], w.ry);
            __stcs(&R.dt[2ull * R.cap + i], w.rz);
            __stcs(&R.vox[R.cap + i], w.iy); // samples
            if (SKIP) { // 1 / direction for the block march
                __stcs(&R.rd[i], w.rdx);
                __stcs(&R.rd[R.cap + i], w.rdy);
                __stcs(&R.rd[2ull * R.cap + i], w.rdz);
            }
            R.flags[i] = (uint8_t)(64 | 128);
            store_mu(R, i, tab);
            continue;
        }
        __stcs(&R.tn[i], w.tnx);
        __stcs(&R.tn[R.cap + i], w.tny);
        __stcs(&R.tn[2ull * R.cap + i], w.tnz);
        __stcs(&R.dt[i], w.dtx);
        __stcs(&R.dt[R.cap + i], w.dty);
        __stcs(&R.dt[2ull * R.cap + i], w.dtz);
        if (SKIP) {
            __stcs(&R.rd[i], w.rdx);
            __stcs(&R.rd[R.cap + i], w.rdy);
            __stcs(&R.rd[2ull * R.cap + i], w.rdz);
        }
        __stcs(&R.vox[i], w.ix);
        __stcs(&R.vox[R.cap + i], w.iy);
        __stcs(&R.vox[2ull * R.cap + i], w.iz);
        R.flags[i] = (uint8_t)((w.sx + 1) | ((w.sy + 1) << 2) | ((w.sz + 1) << 4) | 64);
        store_mu(R, i, tab);
    }
    c_rays = __reduce_add_sync(kFull, c_rays);
    if ((threadIdx.x & 31) == 0 && c_rays)
        red_add(P.accum + P.off_diag + 3, c_rays);
}

// -------------------------------------------------------------------- walk
constexpr int walk_min_blocks(int fmt, bool skip, bool march)
{
    return !skip ? XSW_EXACT_BLOCKS : (fmt == kFmtP8 && !march ? XSW_WALK_BLOCKS : 6);
}

template <int FMT, bool REG, bool SKIP, bool MARCH, int RUN>
__global__ void __launch_bounds__(kBlock, walk_min_blocks(FMT, SKIP, MARCH)) wave_walk(const __grid_constant__ TransportParams P,
                                                    const __grid_constant__ WaveArgs A)
{
    extern __shared__ __align__(16) unsigned char smem[];
    WaveCtl* ctl = A.ctl;
    const WaveRays& R = A.R;
    const uint32_t n = ctl->n_rays, n_s = ctl->n_score;
    const int lane = threadIdx.x & 31;
    const unsigned lt_mask = (1u << lane) - 1u;
    const Grid& G = P.G;
    MuTab<FMT, REG, REG && XSW_WALK_MU_SMEM> tab;
    tab.T = reinterpret_cast<double*>(smem) + threadIdx.x;
    tab.energy = -1.0;
    Walk w;
    w.march = 0;
    bool walking = false, drained = false;
    uint32_t ray = 0;
    // launch counters (free-path / scoring visits, iterations, uniform-block
    // iterations) in shared memory, added when a ray ends: per-lane counter
    // registers would push the loop past the 80-register budget
    __shared__ unsigned int cnt[4];
    if (threadIdx.x < 4)
        cnt[threadIdx.x] = 0u;
    unsigned long long* diag = P.accum + P.off_diag;
    constexpr int kCntSlot[4] = {0, 1, 5, 7}; // diag words: free-path visits, scoring visits, iterations, uniform
    // u32 counters (64-bit shared atomics are CAS loops: +12% walk time); a
    // counter that passes 2^31 is moved to the global u64 word right away
    auto count = [&](int k, uint32_t v) {
        const uint32_t old = atomicAdd(&cnt[k], v);
        if (old + v >= (1u << 31))
            red_add(diag + kCntSlot[k], atomicExch(&cnt[k], 0u));
    };
    __syncthreads();
    uint32_t c_wit = 0;
    // A lane that ends its ray keeps the result in its walker registers until
    // the warp next refills (or the loop ends): the stores then run once per
    // refill instead of in a divergent branch of almost every iteration.
    bool has_result = false;
    auto store_result = [&]() {
        const bool score = ray < n_s;
        if (score) {
            __stcs(&R.res[ray], w.depth);
        } else {
            const bool hit = w.hit != 0;
            __stcs(&R.res[ray], hit ? hit_t(w) : 0.0);
            R.res_hit[ray] = hit ? 1 : 0;
            __stcs(&R.res_vox[ray], w.ix);
            __stcs(&R.res_vox[R.cap + ray], w.iy);
            __stcs(&R.res_vox[2ull * R.cap + ray], w.iz);
        }
        count(score ? 1 : 0, w.steps + w.skipped);
        count(2, w.steps);
        if (w.ucells)
            count(3, w.ucells);
        has_result = false;
    };
    for (;;) {
        const unsigned idle = __ballot_sync(kFull, !walking);
        if (!drained && (idle == kFull || __popc(idle) >= (SKIP ? kRefill : XSW_REFILL_EXACT))) {
            if (has_result)
                store_result();
            uint32_t base = 0;
            if (lane == 0)
                base = atomicAdd(&ctl->cursor, (uint32_t)__popc(idle));
            base = __shfl_sync(kFull, base, 0);
            drained = base + (uint32_t)__popc(idle) >= n;
            if (!walking) {
                const uint32_t r = base + (uint32_t)__popc(idle & lt_mask);
                if (r < n) {
                    const uint8_t f = R.flags[r];
                    if (MARCH && (f & 128)) { // REF trace.cpp:116-134
                        ray = r;
                        w.march = 1;
                        w.t = __ldcs(&R.t[r]);
                        w.texit = __ldcs(&R.texit[r]);
                        w.target = __ldcs(&R.target[r]);
                        w.ox = __ldcs(&R.tn[r]);
                        w.oy = __ldcs(&R.tn[R.cap + r]);
                        w.oz = __ldcs(&R.tn[2ull * R.cap + r]);
                        w.rx = __ldcs(&R.dt[r]);
                        w.ry = __ldcs(&R.dt[R.cap + r]);
                        w.rz = __ldcs(&R.dt[2ull * R.cap + r]);
                        w.ix = 0;
                        w.iy = __ldcs(&R.vox[R.cap + r]);
                        w.dtx = P.march_h;
                        if (SKIP) {
                            w.rdx = __ldcs(&R.rd[r]);
                            w.rdy = __ldcs(&R.rd[R.cap + r]);
                            w.rdz = __ldcs(&R.rd[2ull * R.cap + r]);
                        }
                        load_mu(R, r, tab);
                        w.depth = 0.0;
                        w.hit = 0;
                        w.steps = 0;
                        w.skipped = 0;
                        w.ucells = 0;
                        walking = true;
                    } else if (f & 64) {
                        ray = r;
                        if (MARCH)
                            w.march = 0;
                        w.t = __ldcs(&R.t[r]);
                        w.texit = __ldcs(&R.texit[r]);
                        w.target = __ldcs(&R.target[r]);
                        w.tnx = __ldcs(&R.tn[r]);
                        w.tny = __ldcs(&R.tn[R.cap + r]);
                        w.tnz = __ldcs(&R.tn[2ull * R.cap + r]);
                        w.dtx = __ldcs(&R.dt[r]);
                        w.dty = __ldcs(&R.dt[R.cap + r]);
                        w.dtz = __ldcs(&R.dt[2ull * R.cap + r]);
                        if (SKIP) {
                            w.rdx = __ldcs(&R.rd[r]);
                            w.rdy = __ldcs(&R.rd[R.cap + r]);
                            w.rdz = __ldcs(&R.rd[2ull * R.cap + r]);
                        }
                        w.ix = __ldcs(&R.vox[r]);
                        w.iy = __ldcs(&R.vox[R.cap + r]);
                        w.iz = __ldcs(&R.vox[2ull * R.cap + r]);
                        w.sx = (int)(f & 3) - 1;
                        w.sy = (int)((f >> 2) & 3) - 1;
                        w.sz = (int)((f >> 4) & 3) - 1;
                        w.ax = term_x(G, w.ix);
                        w.ay = term_y(G, w.iy);
                        w.az = term_z(G, w.iz);
                        prefetch<FMT>(G, w.ax + w.ay + w.az, w.raw, w.shift, w.dens);
                        load_mu(R, r, tab);
                        w.depth = 0.0;
                        w.hit = 0;
                        w.steps = 0;
                        w.skipped = 0;
                        w.ucells = 0;
                        walking = true;
                    }
                }
            }
        }
        if (__ballot_sync(kFull, walking) == 0) {
            if (drained)
                break;
            continue;
        }
        // lane slots: the steps a full trip takes (an exact count -- the
        // warp's longest trip -- costs a warp reduction per trip, +5% walk time)
        c_wit += SKIP ? XSW_INNER : 2;
        if (walking) {
            walking = walk_step<FMT, REG, SKIP, RUN, REG && XSW_WALK_MU_SMEM>(P, tab, w);
            ++w.steps;
            // the voxel walk takes a second step per loop trip (halves the per-step
            // loop overhead: -21% walk time on speckled phantoms); the block walk
            // up to XSW_INNER steps between the warp's refill checks
            if (!SKIP && walking) {
                walking = walk_step<FMT, REG, SKIP, RUN, REG && XSW_WALK_MU_SMEM>(P, tab, w);
                ++w.steps;
            }
#pragma unroll 1
            for (int j = 1; j < (SKIP ? XSW_INNER : 1) && walking; ++j) {
                walking = walk_step<FMT, REG, SKIP, RUN, REG && XSW_WALK_MU_SMEM>(P, tab, w);
                ++w.steps;
            }
            has_result = !walking;
        }
    }
    if (has_result)
        store_result();
    if (lane == 0)
        red_add(diag + 6, 32ull * c_wit);
    __syncthreads();
    if (threadIdx.x < 4)
        red_add(diag + kCntSlot[threadIdx.x], cnt[threadIdx.x]);
}

// ---------------------------------------------------------------- complete
// Scoring rays (REF run_history :178-193).  Warp-sized chunks: a history's
// scoring rays sit next to each other in the queue, so a warp folds its
// lanes' scores per slot (exact integer limb sums) and touches each slot's
// total and pending count once.

__global__ void __launch_bounds__(kBlock, XSW_SCORE_MINB) wave_score(const __grid_constant__ TransportParams P,
                                                     const __grid_constant__ WaveArgs A)
{
    extern __shared__ __align__(16) unsigned long long acc[];
    WaveCtl* ctl = A.ctl;
    const WaveQueue& in = ctl->q[A.cur];
    const uint32_t n_s = ctl->n_score;
    const Block B = block_stats(P, acc);
    const WaveRays& R = A.R;
    DevStatus* st = P.status;
    const int lane = threadIdx.x & 31;
    const uint32_t n_warps = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t base = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32u; base < n_s;
         base += n_warps * 32u) {
        const uint32_t i = base + (uint32_t)lane;
        int s = -1;
        uint64_t l0 = 0, l1 = 0, l2 = 0;
        const bool is_score = i < n_s && XS_GUARD(batch_at(in, i / (uint32_t)P.splitting).slot < A.n_slots, st, 13.0);
        if (is_score) {
            s = (int)batch_at(in, i / (uint32_t)P.splitting).slot;
            const uint32_t pix = __ldcs(&R.pix[i]);
            const double x = __ldcs(&R.pre[i]) * nl_exp(-__ldcs(&R.res[i]));
            if (!isfinite(x)) {
                raise(st, XS_E_RUNTIME, kErrNonFinite, A.slots[s].bin, A.slots[s].e_in, x);
            } else if (!quantize(ldexp(x, -P.log2_img), l0, l1, l2)) {
                raise(st, XS_E_RUNTIME, kErrTallyOverflow, A.slots[s].bin, A.slots[s].e_in, x);
                l0 = l1 = l2 = 0;
            } else {
                unsigned long long* img = P.accum + P.off_image + 4ull * pix;
                red_add(img + 0, l0);
                red_add(img + 1, l1);
                red_add(img + 2, l2);
            }
            if (P.track_var) {
                Slot& S = A.slots[s];
                const int k = atomicAdd(&S.n_var, 1);
                if (k < P.var_cap) {
                    P.var_pix[var_base_of(P, s) + k] = pix;
                    P.var_val[var_base_of(P, s) + k] = x;
                }
            }
        }
        const unsigned grp = __match_any_sync(kFull, s);
        // limbs are < 2^32: sum their 16-bit halves exactly in 32 bits
        const uint32_t a0 = __reduce_add_sync(grp, (uint32_t)(l0 & 0xFFFFu));
        const uint32_t b0 = __reduce_add_sync(grp, (uint32_t)(l0 >> 16));
        const uint32_t a1 = __reduce_add_sync(grp, (uint32_t)(l1 & 0xFFFFu));
        const uint32_t b1 = __reduce_add_sync(grp, (uint32_t)(l1 >> 16));
        const uint32_t a2 = __reduce_add_sync(grp, (uint32_t)(l2 & 0xFFFFu));
        const uint32_t b2 = __reduce_add_sync(grp, (uint32_t)(l2 >> 16));
        if (is_score && lane == __ffs(grp) - 1) {
            Slot& S = A.slots[s];
            sadd(&S.T[0], ((uint64_t)b0 << 16) + a0);
            sadd(&S.T[1], ((uint64_t)b1 << 16) + a1);
            sadd(&S.T[2], ((uint64_t)b2 << 16) + a2);
            // the last count-down hands the history to this wave's event
            // kernel, which finalizes it: the kernel boundary orders every
            // warp's tallies and scratch before it, so no fence is needed here
            // (an acquire/release hand-off in this kernel cost 39% of its stall
            // samples in memory barriers)
            if (atomicSub(&S.pending, __popc(grp)) == __popc(grp)) {
                const uint32_t k = atomicAdd(&ctl->n_fin, 1u);
                if (XS_GUARD(k < A.n_slots, st, 19.0))
                    ctl->fin[k] = (uint32_t)s;
            }
        }
    }
    flush_stats(P, B);
}

// Free paths: the history's event (REF run_history :141-223), which pushes
// the next wave's scoring rays and free path.
template <int FMT>
__global__ void __launch_bounds__(kBlock, XSW_EVENT_MINB) wave_event(const __grid_constant__ TransportParams P,
                                                     const __grid_constant__ WaveArgs A)
{
    extern __shared__ __align__(16) unsigned long long acc[];
    WaveCtl* ctl = A.ctl;
    const WaveQueue& in = ctl->q[A.cur];
    const uint32_t n = ctl->n_rays, n_s = ctl->n_score;
    const Block B = block_stats(P, acc);
    Deferred def;
    deferred_reset(def);
    const GlobalQ qs{A.slots, ctl, A.cur ^ 1, -1, &def};
    const WaveRays& R = A.R;
    uint32_t c_int = 0;
    const int lane = threadIdx.x & 31;
    const unsigned lt_mask = (1u << lane) - 1u;
    { // histories the scoring kernel ended: finalize and release (REF run_history :225-241)
        const uint32_t n_fin = ctl->n_fin, n_warps = (gridDim.x * blockDim.x) >> 5;
        for (uint32_t b = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32u; b < n_fin; b += n_warps * 32u) {
            const uint32_t k = b + (uint32_t)lane;
            if (k < n_fin) {
                const int s = (int)ctl->fin[k];
                if (XS_GUARD((uint32_t)s < A.n_slots, P.status, 20.0))
                    finalize_history(P, B, qs, s, var_base_of(P, s), P.status);
            }
            __syncwarp();
            flush_deferred(P, B, ctl, A.cur ^ 1, def, A.n_slots, P.status);
        }
    }
    // Escapes and interactions are gathered per warp: escapes end their
    // histories 32 at a time, the interactions' selection phase (event_select)
    // runs 32 at a time, and its Compton and Rayleigh continuations are
    // gathered again by kind, so each sampler runs with full warps of its kind.
    __shared__ uint32_t bufs[kBlock / 32][4][64]; // hits (ray index), Compton, Rayleigh, escapes (slot)
    uint32_t* hb = bufs[threadIdx.x >> 5][0];
    uint32_t* cb = bufs[threadIdx.x >> 5][1];
    uint32_t* rb = bufs[threadIdx.x >> 5][2];
    uint32_t* eb = bufs[threadIdx.x >> 5][3];
    uint32_t nb = 0, nc = 0, nr = 0, ne = 0; // warp-uniform fill levels
    // escapes (their histories end here) are gathered per warp too and run 32
    // at a time: with a warp's hits idle beside them they ran at partial
    // occupancy (events 50.8 -> 49.8 ms per C3 projection)
    auto escapes = [&](bool all) { // 32 (or, at the end, all) gathered escapes with full warps
        if (all ? ne == 0 : ne < 32)
            return;
        const uint32_t take = ne < 32 ? ne : 32;
        const uint32_t sl = (uint32_t)lane < take ? eb[ne - take + lane] : 0u;
        __syncwarp();
        ne -= take;
        if ((uint32_t)lane < take)
            event_select<FMT>(P, B, qs, (int)sl, false, 0.0, 0, 0, 0, var_base_of(P, (int)sl), P.status);
        __syncwarp();
        flush_deferred(P, B, ctl, A.cur ^ 1, def, A.n_slots, P.status);
    };
    auto cont = [&](uint32_t* q, uint32_t& n, bool all) { // run 32 (or, at the end, all) continuations
        if (all ? n == 0 : n < 32)
            return;
        const uint32_t take = n < 32 ? n : 32;
        const uint32_t sl = (uint32_t)lane < take ? q[n - take + lane] : 0u;
        __syncwarp();
        n -= take;
        if ((uint32_t)lane < take)
            event_continue(P, B, qs, (int)sl, var_base_of(P, (int)sl), P.status);
        __syncwarp();
        flush_deferred(P, B, ctl, A.cur ^ 1, def, A.n_slots, P.status);
    };
    auto select = [&](bool active, uint32_t i) { // selection phase for the lanes with `active`
        int kind = K_NONE, s = 0;
        if (active) {
            s = (int)in.free[i - n_s];
            const int vx = __ldcs(&R.res_vox[i]), vy = __ldcs(&R.res_vox[R.cap + i]),
                      vz = __ldcs(&R.res_vox[2ull * R.cap + i]);
            if (XS_GUARD((uint32_t)s < A.n_slots && (uint32_t)vx < (uint32_t)P.G.nx && (uint32_t)vy < (uint32_t)P.G.ny &&
                             (uint32_t)vz < (uint32_t)P.G.nz,
                         P.status, 11.0))
                kind = event_select<FMT>(P, B, qs, s, true, __ldcs(&R.res[i]), vx, vy, vz, var_base_of(P, s), P.status);
        }
        __syncwarp();
        flush_deferred(P, B, ctl, A.cur ^ 1, def, A.n_slots, P.status);
        const unsigned mc = __ballot_sync(kFull, kind == K_COMPTON);
        const unsigned mr = __ballot_sync(kFull, kind == K_RAYLEIGH);
        if (kind == K_COMPTON)
            cb[nc + __popc(mc & lt_mask)] = (uint32_t)s;
        if (kind == K_RAYLEIGH)
            rb[nr + __popc(mr & lt_mask)] = (uint32_t)s;
        nc += __popc(mc);
        nr += __popc(mr);
        __syncwarp();
        cont(cb, nc, false);
        cont(rb, nr, false);
    };
    for (uint32_t base = 0, end = 0;; base += 32) {
        if (base >= end) { // 4 warp-chunks per cursor reservation
            if (lane == 0)
                base = atomicAdd(&ctl->ev_cursor, 128u);
            base = __shfl_sync(kFull, base, 0) + n_s;
            end = base + 128u;
        }
        if (base >= n)
            break;
        const uint32_t i = base + (uint32_t)lane;
        const bool valid = i < n;
        const bool hit = valid && R.res_hit[i] != 0;
        { // escapes are gathered too and run 32 at a time (their history ends)
            const int s = valid && !hit ? (int)in.free[i - n_s] : -1;
            const bool esc = s >= 0 && XS_GUARD((uint32_t)s < A.n_slots, P.status, 12.0);
            const unsigned em = __ballot_sync(kFull, esc);
            if (esc)
                eb[ne + __popc(em & lt_mask)] = (uint32_t)s;
            ne += __popc(em);
            __syncwarp();
            escapes(false);
        }
        const unsigned hm = __ballot_sync(kFull, hit);
        if (hit)
            hb[nb + __popc(hm & lt_mask)] = i;
        nb += __popc(hm);
        c_int += hit;
        __syncwarp();
        if (nb >= 32) {
            const uint32_t j = hb[nb - 32 + lane];
            __syncwarp();
            nb -= 32;
            select(true, j);
        }
        __syncwarp();
    }
    if (nb > 0) {
        const uint32_t j = (uint32_t)lane < nb ? hb[lane] : 0u;
        const bool act = (uint32_t)lane < nb;
        __syncwarp();
        nb = 0;
        select(act, j);
    }
    cont(cb, nc, true);
    cont(rb, nr, true);
    escapes(true);
    if (c_int)
        atomicAdd(B.diag + 4, (unsigned long long)c_int);
    flush_stats(P, B);
}

// ------------------------------------------------------------ admission
__global__ void wave_plan(const __grid_constant__ TransportParams P, const __grid_constant__ WaveArgs A)
{
    WaveCtl* ctl = A.ctl;
    const int32_t top = ctl->free_top;
    // claim up to one history per free slot from the shared counter (several
    // pipelines admit concurrently; claims past h_end are simply empty)
    const unsigned long long base = top > 0 ? atomicAdd(A.next_h, (unsigned long long)top) : *A.next_h;
    const unsigned long long left = base < P.h_end ? P.h_end - base : 0ull;
    const uint32_t k = (unsigned long long)top < left ? (uint32_t)top : (uint32_t)left;
    ctl->admit_base = base;
    ctl->admit_n = k;
    ctl->next_h = base + (unsigned long long)top;
    ctl->admit_q = ctl->q[A.cur].n_free; // admitted histories' free paths follow the events'
    ctl->q[A.cur].n_free += k;
    ctl->free_top = top - (int32_t)k; // admitted slots: free_stack[top - k, top)
    ctl->live = A.n_slots - (uint32_t)ctl->free_top;
    ctl->setup_cursor = 0;
    ++ctl->waves;
}

__global__ void __launch_bounds__(kBlock, XSW_ADMIT_MINB) wave_admit(const __grid_constant__ TransportParams P,
                                                     const __grid_constant__ WaveArgs A)
{
    extern __shared__ __align__(16) unsigned long long acc[];
    WaveCtl* ctl = A.ctl;
    const uint32_t k = ctl->admit_n;
    if (k == 0)
        return;
    // the bin search of history_start runs on a shared-memory copy of the
    // bin offsets (after the block statistics)
    uint64_t* sstart = reinterpret_cast<uint64_t*>(acc + stat_words(P.n_bins));
    for (int i = threadIdx.x; i <= P.n_bins; i += blockDim.x)
        sstart[i] = P.bin_start[i];
    const Block B = block_stats(P, acc); // (synchronises)
    const int32_t top = ctl->free_top;
    const unsigned long long base = ctl->admit_base;
    const uint32_t qb = ctl->admit_q;
    Deferred def;
    deferred_reset(def);
    // the histories' initial weights (REF WeightLedger::initial): limb sums in
    // registers, one warp reduction at the end (every admitted history adds to
    // the same three words: shared-memory atomics there serialise)
    unsigned long long w0l[3] = {0ull, 0ull, 0ull};
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t i0 = blockIdx.x * blockDim.x + (threadIdx.x & ~31u); i0 < k; i0 += stride) {
        const uint32_t i = i0 + (threadIdx.x & 31u);
        if (i < k) {
            const int s = (int)ctl->free_stack[top + i];
            const GlobalQ qs{A.slots, ctl, A.cur, (int)(qb + i), &def};
            const double w0 = history_start(P, B, qs, sstart, s, base + i, P.status, false);
            uint64_t l0, l1, l2;
            if (w0 != 0.0) {
                if (quantize(ldexp(w0, -P.log2_w), l0, l1, l2)) {
                    w0l[0] += l0;
                    w0l[1] += l1;
                    w0l[2] += l2;
                } else {
                    raise(P.status, XS_E_RUNTIME, kErrTallyOverflow, 0, 0.0, w0);
                }
            }
        }
        __syncwarp();
        flush_deferred(P, B, ctl, A.cur, def, A.n_slots, P.status);
    }
    for (int j = 0; j < 3; ++j) {
        unsigned long long v = w0l[j];
        for (int o = 16; o > 0; o >>= 1)
            v += __shfl_xor_sync(kFull, v, o);
        if ((threadIdx.x & 31) == 0)
            red_add(P.accum + P.off_ledger + j, v);
    }
    flush_stats(P, B);
}

__global__ void wave_init(WaveCtl* ctl, uint32_t* stack, uint32_t n_slots, unsigned long long h_begin)
{
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n_slots; i += gridDim.x * blockDim.x)
        stack[i] = n_slots - 1 - i;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        ctl->free_top = (int32_t)n_slots;
        ctl->next_h = h_begin; // this pipeline's last view of the shared counter
        ctl->q[0].n_batch = ctl->q[0].n_free = ctl->q[0].n_batch_r = 0;
        ctl->q[1].n_batch = ctl->q[1].n_free = ctl->q[1].n_batch_r = 0;
        ctl->waves = 0;
        ctl->live = 0;
    }
}

bool use_reg_w(const TransportParams& P) { return (P.G.fmt == kFmtP4 || P.G.fmt == kFmtP8) && P.n_pal <= 4; }

typedef void (*WaveFn)(const TransportParams, const WaveArgs);

struct WaveSet {
    WaveFn setup, walk, event;
};

template <int FMT, bool REG, bool SKIP, bool MARCH, int RUN = 0>
WaveSet wave_set()
{
    return {wave_setup<FMT, REG, SKIP, MARCH>, wave_walk<FMT, REG, SKIP, MARCH, RUN>, wave_event<FMT>};
}

// the walk with the run field along x / y (8-bit palette, block walk, the
// walker's exact steps: free paths and scoring rays alike)
template <bool REG>
WaveSet wave_set_runs(const Grid& G)
{
    return G.run_axis == 0 ? wave_set<kFmtP8, REG, true, false, 1>() : wave_set<kFmtP8, REG, true, false, 2>();
}

template <bool MARCH>
WaveSet wave_kernels_m(const TransportParams& P)
{
    const bool skip = P.skip != 0 && P.G.ubit != 0;
    if (P.G.fmt == kFmtP4) {
        if (use_reg_w(P))
            return skip ? wave_set<kFmtP4, true, true, MARCH>() : wave_set<kFmtP4, true, false, MARCH>();
        return skip ? wave_set<kFmtP4, false, true, MARCH>() : wave_set<kFmtP4, false, false, MARCH>();
    }
    if (P.G.fmt == kFmtP8) {
        if (!MARCH && skip && P.G.run_mask)
            return use_reg_w(P) ? wave_set_runs<true>(P.G) : wave_set_runs<false>(P.G);
        if (use_reg_w(P))
            return skip ? wave_set<kFmtP8, true, true, MARCH>() : wave_set<kFmtP8, true, false, MARCH>();
        return skip ? wave_set<kFmtP8, false, true, MARCH>() : wave_set<kFmtP8, false, false, MARCH>();
    }
    return wave_set<kFmtRaw, false, false, MARCH>();
}

WaveSet wave_kernels_for(const TransportParams& P)
{
    return P.step_voxels > 1 ? wave_kernels_m<true>(P) : wave_kernels_m<false>(P);
}

template <class T>
cudaError_t grow(T*& p, size_t& have, size_t need)
{
    if (have >= need)
        return cudaSuccess;
    if (p)
        cudaFree(p);
    p = nullptr;
    have = 0;
    cudaError_t e = cudaMalloc(&p, need * sizeof(T));
    if (e == cudaSuccess)
        have = need;
    return e;
}

} // namespace

// ------------------------------------------------------------------- host
// One pipeline: its histories (slots), queues, ray arrays and stream.  Two
// pipelines run on two streams and share the history counter, so one's
// latency-bound event/set-up kernels overlap the other's issue-bound walk and
// each kernel's tail is filled by the other pipeline's work.
struct WavePipe {
    Slot* slots = nullptr;
    size_t n_slots_have = 0;
    uint32_t* stack = nullptr;
    size_t stack_have = 0;
    WaveCtl* ctl = nullptr;
    size_t ctl_have = 0;
    ScoreBatch* sq[2] = {nullptr, nullptr};
    size_t sq_have[2] = {0, 0};
    uint32_t* fq[2] = {nullptr, nullptr};
    size_t fq_have[2] = {0, 0};
    double* dbl = nullptr; // t, texit, target, tn x3, dt x3, mu x n_mu, pre, res
    size_t dbl_have = 0;
    double* rd = nullptr;
    size_t rd_have = 0;
    int* vox = nullptr; // vox x3, res_vox x3, pix
    size_t vox_have = 0;
    uint8_t* bytes = nullptr; // flags, res_hit
    size_t bytes_have = 0;
    WaveCtl* host_ctl = nullptr; // pinned
    cudaStream_t stream = nullptr;
    cudaEvent_t join = nullptr;
    std::vector<cudaEvent_t> ev; // walk-kernel timing, a pair per wave
    // per run
    WaveArgs A;
    TransportParams P;
    int cur = 0;
    uint32_t waves = 0;     // waves launched in this call (every job)
    uint32_t job_waves = 0; // ... for the current job
    bool done = false;

    size_t bytes_held() const
    {
        return n_slots_have * sizeof(Slot) + stack_have * 4 + (sq_have[0] + sq_have[1]) * sizeof(ScoreBatch) +
               (fq_have[0] + fq_have[1]) * 4 + dbl_have * 8 + rd_have * 8 + vox_have * 4 + bytes_have;
    }
    void release()
    {
        cudaFree(slots);
        cudaFree(stack);
        cudaFree(ctl);
        for (int b = 0; b < 2; ++b) {
            cudaFree(sq[b]);
            cudaFree(fq[b]);
        }
        cudaFree(dbl);
        cudaFree(rd);
        cudaFree(vox);
        cudaFree(bytes);
        if (host_ctl)
            cudaFreeHost(host_ctl);
        for (cudaEvent_t v : ev)
            cudaEventDestroy(v);
        if (join)
            cudaEventDestroy(join);
        if (stream)
            cudaStreamDestroy(stream);
    }
};

constexpr int kMaxPipes = 4;

struct WaveEngine {
    WavePipe pipe[kMaxPipes];
    unsigned long long* next_h = nullptr;
    cudaEvent_t fork = nullptr;
    // the last memory-clamp decision: (requested slots, splitting, n_mu,
    // pipes) -> slots; repeated calls reuse it (the buffers are already held)
    // instead of asking cudaMemGetInfo, which took up to 63 ms per call
    uint64_t clamp_key[4] = {0, 0, 0, 0};
    uint32_t clamp_slots = 0;
};

namespace {

// ---------------------------------------------------------- walk probe
// Does crossing uniform blocks pay on this phantom?  A block step costs about
// 1.7x a voxel step, so on speckled grids (segmented reconstructions: few
// uniform blocks along the rays) the plain voxel walk is faster.  At upload,
// a fixed set of rays (start points in non-vacuum voxels, isotropic
// directions, a counter hash of the ray index: deterministic per phantom) is
// walked to the grid exit in both modes, counting loop iterations.
__device__ __forceinline__ uint32_t probe_hash(uint32_t x)
{
    x ^= x >> 16;
    x *= 0x7FEB352Du;
    x ^= x >> 15;
    x *= 0x846CA68Bu;
    x ^= x >> 16;
    return x;
}
__device__ __forceinline__ double probe_u(uint32_t i, uint32_t k)
{
    return (probe_hash(i * 0x9E3779B9u + k * 0x85EBCA6Bu + 0x1234567u) >> 8) * (1.0 / 16777216.0) + 0.5 / 16777216.0;
}

template <int FMT, bool SKIP>
__global__ void __launch_bounds__(kBlock) walk_probe(const __grid_constant__ TransportParams P, int n_rays,
                                                     unsigned long long* iters)
{
    const Grid& G = P.G;
    MuTab<FMT, true> tab;
    tab.t0 = tab.t1 = tab.t2 = tab.t3 = 1.0;
    tab.T = nullptr;
    tab.energy = 0.0;
    unsigned long long n_it = 0;
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n_rays; r += gridDim.x * blockDim.x) {
        V3 o = v3(0.0, 0.0, 0.0);
        for (int k = 0; k < 8; ++k) { // a point in matter (last try kept)
            o = v3(G.ox + probe_u(r, 3 * k) * (G.ux - G.ox), G.oy + probe_u(r, 3 * k + 1) * (G.uy - G.oy),
                   G.oz + probe_u(r, 3 * k + 2) * (G.uz - G.oz));
            int code;
            float dens = 0.f;
            fetch<FMT>(G, voxel_of(o.x, G.ox, G.ihx, G.nx), voxel_of(o.y, G.oy, G.ihy, G.ny),
                       voxel_of(o.z, G.oz, G.ihz, G.nz), code, dens);
            if (P.pal_mat[(code & ~G.ubit) & (kMaxPalette - 1)] != 0)
                break;
        }
        const double cz = 2.0 * probe_u(r, 40) - 1.0, ph = 6.283185307179586 * probe_u(r, 41);
        const double sz = sqrt(fmax(0.0, 1.0 - cz * cz));
        const V3 d = v3(sz * cos(ph), sz * sin(ph), cz);
        Walk w;
        w.march = 0;
        if (!walk_begin<FMT, SKIP>(P, w, o, d, CUDART_INF, false, nullptr, 0))
            continue;
        bool walking = true;
        while (walking) {
            walking = walk_step<FMT, true, SKIP, 0>(P, tab, w);
            ++n_it;
        }
    }
    n_it = __reduce_add_sync(kFull, (unsigned)n_it);
    if ((threadIdx.x & 31) == 0)
        atomicAdd(iters, n_it);
}

} // namespace

// iters[0]: voxel-walk iterations, iters[1]: block-walk iterations (device, zeroed here)
cudaError_t launch_walk_probe(const TransportParams& P, unsigned long long* iters, cudaStream_t s)
{
    cudaError_t e = cudaMemsetAsync(iters, 0, 2 * sizeof(unsigned long long), s);
    if (e != cudaSuccess)
        return e;
    const int n = 8192, grid = (n + kBlock - 1) / kBlock;
    if (P.G.fmt == kFmtP4) {
        walk_probe<kFmtP4, false><<<grid, kBlock, 0, s>>>(P, n, iters);
        walk_probe<kFmtP4, true><<<grid, kBlock, 0, s>>>(P, n, iters + 1);
    } else {
        walk_probe<kFmtP8, false><<<grid, kBlock, 0, s>>>(P, n, iters);
        walk_probe<kFmtP8, true><<<grid, kBlock, 0, s>>>(P, n, iters + 1);
    }
    return cudaGetLastError();
}

WaveEngine* wave_create() { return new WaveEngine(); }

void wave_destroy(WaveEngine* e)
{
    if (!e)
        return;
    for (WavePipe& p : e->pipe)
        p.release();
    cudaFree(e->next_h);
    if (e->fork)
        cudaEventDestroy(e->fork);
    delete e;
}

size_t wave_slot_bytes() { return sizeof(Slot); }

#ifdef XSW_DEBUG_SYNC
#define XSW_CHECK(x)                                                                               \
    do {                                                                                           \
        cudaError_t err_ = (x);                                                                    \
        if (err_ != cudaSuccess) {                                                                 \
            std::fprintf(stderr, "XSW_CHECK failed at wavefront.cu:%d: %s\n", __LINE__,           \
                         cudaGetErrorString(err_));                                                \
            return err_;                                                                           \
        }                                                                                          \
    } while (0)
#else
#define XSW_CHECK(x)                                                                               \
    do {                                                                                           \
        cudaError_t err_ = (x);                                                                    \
        if (err_ != cudaSuccess)                                                                   \
            return err_;                                                                           \
    } while (0)
#endif

// Device bytes of one pipeline with n_slots live histories (pipe_prepare).
static double pipe_bytes(uint32_t n_slots, int splitting, int n_mu)
{
    const double cap = (double)n_slots * ((double)splitting + 1.0);
    const double per_ray = (3 + 3 + 3 + n_mu + 2) * 8.0 + 3 * 8.0 + 7 * 4.0 + 2.0;
    const double per_slot = (double)sizeof(Slot) + 8.0 + 2.0 * (sizeof(ScoreBatch) + 4.0);
    return cap * per_ray + (double)n_slots * per_slot;
}

static cudaError_t pipe_prepare(WavePipe& w, const TransportParams& P, uint32_t n_slots, int n_mu)
{
    const uint64_t split = (uint64_t)P.splitting;
    const uint64_t cap = (uint64_t)n_slots * (split + 1);
    if (cap >= (1ull << 32))
        return cudaErrorInvalidValue;
    XSW_CHECK(grow(w.slots, w.n_slots_have, n_slots));
    XSW_CHECK(grow(w.stack, w.stack_have, 2 * (size_t)n_slots)); // free stack | finalize list
    XSW_CHECK(grow(w.ctl, w.ctl_have, 1));
    for (int b = 0; b < 2; ++b) {
        XSW_CHECK(grow(w.sq[b], w.sq_have[b], (size_t)n_slots));
        XSW_CHECK(grow(w.fq[b], w.fq_have[b], (size_t)n_slots));
    }
    const size_t n_dbl = (size_t)(3 + 3 + 3 + n_mu + 2);
    XSW_CHECK(grow(w.dbl, w.dbl_have, n_dbl * cap));
    XSW_CHECK(grow(w.rd, w.rd_have, 3 * cap));
    XSW_CHECK(grow(w.vox, w.vox_have, 7 * cap));
    XSW_CHECK(grow(w.bytes, w.bytes_have, 2 * cap));
    if (!w.host_ctl)
        XSW_CHECK(cudaHostAlloc(&w.host_ctl, sizeof(WaveCtl), cudaHostAllocDefault));
    if (!w.stream)
        XSW_CHECK(cudaStreamCreateWithFlags(&w.stream, cudaStreamNonBlocking));
    if (!w.join)
        XSW_CHECK(cudaEventCreateWithFlags(&w.join, cudaEventDisableTiming));

    WaveArgs& A = w.A;
    std::memset(&A, 0, sizeof A);
    A.slots = w.slots;
    A.ctl = w.ctl;
    A.n_slots = n_slots;
    WaveRays& R = A.R;
    R.cap = (uint32_t)cap;
    R.n_mu = n_mu;
    double* d = w.dbl;
    R.t = d;
    R.texit = d + cap;
    R.target = d + 2 * cap;
    R.tn = d + 3 * cap;
    R.dt = d + 6 * cap;
    R.mu = d + 9 * cap;
    R.pre = d + (9 + n_mu) * cap;
    R.res = d + (10 + n_mu) * cap;
    R.rd = w.rd;
    R.vox = w.vox;
    R.res_vox = w.vox + 3 * cap;
    R.pix = reinterpret_cast<uint32_t*>(w.vox + 6 * cap);
    R.flags = w.bytes;
    R.res_hit = w.bytes + cap;
    return cudaSuccess;
}

// jobs: one projection (n_jobs = 1: its histories shared by every pipeline
// through one counter), or several projections of the same scene, run field,
// palette and sizes that differ only in angle, accumulator and status (a scan):
// each pipeline then runs one job at a time with its own counter and takes the
// next job as soon as its current one has drained, so one projection's ramp-down
// overlaps the other pipelines' steady state.
cudaError_t wave_run_jobs(WaveEngine* e, const TransportParams* jobs, int n_jobs, int sm_count, uint32_t n_slots,
                          cudaStream_t s, WaveInfo* info, cudaEvent_t start, int n_pipes)
{
    const auto host_t0 = std::chrono::steady_clock::now();
    const TransportParams& P = jobs[0];
    const bool multi = n_jobs > 1;
    const uint64_t n_hist = P.h_end - P.h_begin;
    if (n_slots > n_hist)
        n_slots = (uint32_t)n_hist;
    if (n_slots < 1)
        n_slots = 1;
    n_pipes = n_pipes < 1 ? 1 : (n_pipes > kMaxPipes ? kMaxPipes : n_pipes);
    if (n_slots < 2)
        n_pipes = 1;
    if (multi && n_pipes > n_jobs)
        n_pipes = n_jobs;
    // per-lane mu table entries: palette codes (4-bit palette, up to 16) or
    // materials (8-bit palette / raw ids, up to kMaxMaterials)
    const int n_mu = use_reg_w(P) ? 4 : (P.G.fmt == kFmtP4 ? std::max(P.n_pal, 1) : kMaxMaterials);
    const uint64_t key[4] = {n_slots, (uint64_t)P.splitting, (uint64_t)n_mu, (uint64_t)n_pipes};
    if (e->clamp_slots && std::equal(key, key + 4, e->clamp_key)) {
        n_slots = e->clamp_slots;
    } else { // live histories are bounded by device memory: the walker state grows
      // with splitting (n_slots * (splitting + 1) ray entries), so a large
      // splitting factor gets fewer slots instead of failing the run
        size_t free_b = 0, total_b = 0;
        if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess) {
            size_t held = 0;
            for (const WavePipe& w : e->pipe)
                held += w.bytes_held();
            const double budget = 0.7 * (double)(free_b + held);
            while (n_slots > 4096 && (double)n_pipes * pipe_bytes((n_slots + n_pipes - 1) / n_pipes, P.splitting, n_mu) > budget)
                n_slots >>= 1;
        }
        std::copy(key, key + 4, e->clamp_key);
        e->clamp_slots = n_slots;
    }
    const auto host_ta = std::chrono::steady_clock::now();
    const uint32_t per = (n_slots + n_pipes - 1) / n_pipes;
    for (int p = 0; p < n_pipes; ++p) {
        WavePipe& w = e->pipe[p];
        XSW_CHECK(pipe_prepare(w, P, per, n_mu));
        w.waves = 0;
    }
    const auto host_tb = std::chrono::steady_clock::now();
    if (!e->next_h) // history counters: one per pipeline (jobs), the first shared (one projection)
        XSW_CHECK(cudaMalloc(&e->next_h, kMaxPipes * sizeof(unsigned long long)));
    if (!e->fork)
        XSW_CHECK(cudaEventCreateWithFlags(&e->fork, cudaEventDisableTiming));

    const WaveSet K = wave_kernels_for(P);
    const size_t mu_smem = use_reg_w(P) ? 0 : (size_t)n_mu * kBlock * 8;
    const size_t walk_smem = use_reg_w(P) ? (XSW_WALK_MU_SMEM ? (size_t)4 * kBlock * 8 : 0) : mu_smem;
    const size_t stat_smem = stat_words(P.n_bins) * 8;
    XSW_CHECK(cudaFuncSetAttribute((const void*)K.setup, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)std::max<size_t>(mu_smem, 1)));
    XSW_CHECK(cudaFuncSetAttribute((const void*)K.walk, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)std::max<size_t>(walk_smem, 1)));
    XSW_CHECK(cudaFuncSetAttribute((const void*)K.event, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)stat_smem));
    XSW_CHECK(cudaFuncSetAttribute((const void*)wave_score, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)stat_smem));
    const size_t admit_smem = stat_smem + (size_t)(P.n_bins + 1) * 8;
    XSW_CHECK(cudaFuncSetAttribute((const void*)wave_admit, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)admit_smem));
    int walk_per_sm = 0;
    XSW_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&walk_per_sm, K.walk, kBlock, walk_smem));
    if (walk_per_sm < 1)
        walk_per_sm = 1;
    int walk_use = walk_per_sm;
    if (const char* v = std::getenv("XSCAT_WALK_BPS")) // experiment: walk blocks per SM actually launched
        walk_use = std::max(1, std::min(walk_per_sm, std::atoi(v)));
    const int g_walk = sm_count * walk_use;
    // grid-stride kernels: as many resident blocks as fit (they are latency-bound)
    auto resident = [&](const void* k, size_t smem, int* out) -> cudaError_t {
        int per = 0;
        cudaError_t err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, kBlock, smem);
        *out = sm_count * (per < 1 ? 1 : per);
        return err;
    };
    int g_work = 0, g_setup = 0, g_score = 0, g_admit = 0;
    XSW_CHECK(resident((const void*)K.event, stat_smem, &g_work));
    XSW_CHECK(resident((const void*)K.setup, mu_smem, &g_setup));
    XSW_CHECK(resident((const void*)wave_score, stat_smem, &g_score));
    XSW_CHECK(resident((const void*)wave_admit, admit_smem, &g_admit));

    const auto host_t1 = std::chrono::steady_clock::now();
    if (start) // buffers are allocated: the timed region starts here
        XSW_CHECK(cudaEventRecord(start, s));
    if (!multi)
        XSW_CHECK(cudaMemcpyAsync(e->next_h, &P.h_begin, sizeof(unsigned long long), cudaMemcpyHostToDevice, s));
    XSW_CHECK(cudaEventRecord(e->fork, s));
    uint32_t launches = 0;
    // start job j on pipeline p (its stream is ordered after the fork)
    auto start_job = [&](int p, int j) -> cudaError_t {
        WavePipe& w = e->pipe[p];
        cudaStream_t ps = w.stream;
        w.P = jobs[j];
        if (w.P.track_var) { // scratch: var_cap entries per slot, pipelines side by side
            w.P.var_pix = jobs[j].var_pix + (size_t)p * per * jobs[j].var_cap;
            w.P.var_val = jobs[j].var_val + (size_t)p * per * jobs[j].var_cap;
        }
        unsigned long long* cnt = multi ? e->next_h + p : e->next_h;
        if (multi)
            XSW_CHECK(cudaMemcpyAsync(cnt, &jobs[j].h_begin, sizeof(unsigned long long), cudaMemcpyHostToDevice, ps));
        WaveCtl init;
        std::memset(&init, 0, sizeof init);
        for (int b = 0; b < 2; ++b) {
            init.q[b].batch = w.sq[b];
            init.q[b].cap = per;
            init.q[b].free = w.fq[b];
        }
        init.free_stack = w.stack;
        init.fin = w.stack + per;
        XSW_CHECK(cudaMemcpyAsync(w.ctl, &init, sizeof init, cudaMemcpyHostToDevice, ps));
        wave_init<<<sm_count, 256, 0, ps>>>(w.ctl, w.stack, per, jobs[j].h_begin);
        w.A.next_h = cnt;
        w.cur = 0;
        w.job_waves = 0;
        w.done = false;
        w.A.cur = 0;
        wave_plan<<<1, 1, 0, ps>>>(w.P, w.A);
        wave_admit<<<g_admit, kBlock, admit_smem, ps>>>(w.P, w.A);
        XSW_CHECK(cudaGetLastError());
        launches += 3;
        return cudaSuccess;
    };
    int next_job = 0;
    for (int p = 0; p < n_pipes; ++p) {
        XSW_CHECK(cudaStreamWaitEvent(e->pipe[p].stream, e->fork, 0));
        XSW_CHECK(start_job(p, multi ? next_job++ : 0));
    }
    // XSCAT_KTIME=1: CUDA events around every kernel of the wave (per-kernel
    // device time in xs_launch_stats; meaningful with one pipeline)
    const bool ktime = std::getenv("XSCAT_KTIME") != nullptr;
    const int kEv = ktime ? 6 : 2;
    int check_every = 4;
    if (const char* v = std::getenv("XSCAT_CHECK_EVERY")) // experiment: waves between host checks
        check_every = std::max(1, std::min(64, std::atoi(v)));
    const xsi::Range range("xscat: wavefront waves");
    for (;;) {
        for (int k = 0; k < check_every; ++k)
            for (int p = 0; p < n_pipes; ++p) {
                WavePipe& w = e->pipe[p];
                if (w.done)
                    continue;
                cudaStream_t ps = w.stream;
                WaveArgs& A = w.A;
                while (w.ev.size() < (size_t)kEv * (size_t)(w.waves + 1)) {
                    cudaEvent_t v;
                    XSW_CHECK(cudaEventCreate(&v));
                    w.ev.push_back(v);
                }
                A.cur = w.cur;
#ifdef XSW_DEBUG_SYNC // debugging aid: name the kernel that faults (host-side only)
                auto dbg_wait = [&](const char* what) {
                    const cudaError_t err = cudaStreamSynchronize(ps);
                    if (err != cudaSuccess) {
                        std::fprintf(stderr, "FAULT in %s, pipe %d wave %u: %s\n", what, p, w.waves, cudaGetErrorString(err));
                        std::fflush(stderr);
                        _exit(3);
                    }
                };
#else
                auto dbg_wait = [](const char*) {};
#endif
                cudaEvent_t* ev = &w.ev[(size_t)kEv * w.waves]; // [walk start, walk end(, ...)]
                if (ktime)
                    XSW_CHECK(cudaEventRecord(ev[2], ps));
                K.setup<<<g_setup, kBlock, mu_smem, ps>>>(w.P, A);
                dbg_wait("setup");
                XSW_CHECK(cudaEventRecord(ev[0], ps));
                K.walk<<<g_walk, kBlock, walk_smem, ps>>>(w.P, A);
                dbg_wait("walk");
                XSW_CHECK(cudaEventRecord(ev[1], ps));
                wave_score<<<g_score, kBlock, stat_smem, ps>>>(w.P, A);
                dbg_wait("score");
                if (ktime)
                    XSW_CHECK(cudaEventRecord(ev[3], ps));
                K.event<<<g_work, kBlock, stat_smem, ps>>>(w.P, A);
                dbg_wait("event");
                if (ktime)
                    XSW_CHECK(cudaEventRecord(ev[4], ps));
                A.cur = w.cur ^ 1;
                wave_plan<<<1, 1, 0, ps>>>(w.P, A);
                wave_admit<<<g_admit, kBlock, admit_smem, ps>>>(w.P, A);
                dbg_wait("admit");
                if (ktime)
                    XSW_CHECK(cudaEventRecord(ev[5], ps));
                w.cur ^= 1;
                ++w.waves;
                ++w.job_waves;
                launches += 6;
            }
        XSW_CHECK(cudaGetLastError());
        for (int p = 0; p < n_pipes; ++p) {
            WavePipe& w = e->pipe[p];
            if (!w.done)
                XSW_CHECK(cudaMemcpyAsync(w.host_ctl, w.ctl, sizeof(WaveCtl), cudaMemcpyDeviceToHost, w.stream));
        }
        DevStatus hs[kMaxPipes]; // (jobs may share one status record)
        for (int p = 0; p < n_pipes; ++p) {
            hs[p].code = 0;
            if (!e->pipe[p].done) // (read after the stream synchronize below)
                XSW_CHECK(cudaMemcpyAsync(&hs[p], e->pipe[p].P.status, sizeof(DevStatus), cudaMemcpyDeviceToHost,
                                          e->pipe[p].stream));
        }
        bool all_done = true;
        for (int p = 0; p < n_pipes; ++p) {
            WavePipe& w = e->pipe[p];
            if (w.done)
                continue;
            XSW_CHECK(cudaStreamSynchronize(w.stream));
            const WaveCtl& h = *w.host_ctl;
            // nothing left to admit (the shared counter, as this pipeline last saw it,
            // is past the end) and no history in flight
            w.done = h.live == 0 && h.next_h >= w.P.h_end && h.q[w.cur].n_batch == 0 && h.q[w.cur].n_batch_r == 0 &&
                     h.q[w.cur].n_free == 0;
        }
        bool failed = false;
        for (int p = 0; p < n_pipes; ++p)
            failed = failed || hs[p].code != 0;
        if (failed)
            break;
        for (int p = 0; p < n_pipes; ++p) { // a drained pipeline takes the next job
            WavePipe& w = e->pipe[p];
            if (w.done && multi && next_job < n_jobs)
                XSW_CHECK(start_job(p, next_job++));
            all_done = all_done && w.done;
        }
        if (all_done)
            break;
        // every wave advances each live history by one free path: a history
        // needs at most max_interactions + 1 of them, so the run cannot need
        // more waves than this unless the pipeline state is corrupt
        uint32_t max_w = 0;
        for (int p = 0; p < n_pipes; ++p)
            max_w = std::max(max_w, e->pipe[p].job_waves);
        const uint64_t bound = 4ull * ((n_hist + n_slots - 1) / n_slots + 1) * (uint64_t)(P.max_inter + 2) + 64;
        if (max_w > bound) {
            DevStatus bad{};
            bad.code = XS_E_RUNTIME;
            bad.what = kErrStuck;
            for (int p = 0; p < n_pipes; ++p)
                XSW_CHECK(cudaMemcpyAsync(e->pipe[p].P.status, &bad, sizeof bad, cudaMemcpyHostToDevice,
                                          e->pipe[p].stream));
            break;
        }
    }
    const auto host_t2 = std::chrono::steady_clock::now();
    uint32_t waves = 0;
    float walk = 0.f;
    for (int p = 0; p < n_pipes; ++p) {
        WavePipe& w = e->pipe[p];
        XSW_CHECK(cudaEventRecord(w.join, w.stream));
        XSW_CHECK(cudaStreamWaitEvent(s, w.join, 0));
        XSW_CHECK(cudaStreamSynchronize(w.stream));
        for (uint32_t i = 0; i < w.waves; ++i) {
            const cudaEvent_t* ev = &w.ev[(size_t)kEv * i];
            float ms = 0.f;
            XSW_CHECK(cudaEventElapsedTime(&ms, ev[0], ev[1]));
            walk += ms;
            if (ktime && info) {
                XSW_CHECK(cudaEventElapsedTime(&ms, ev[2], ev[0]));
                info->setup_ms += ms;
                XSW_CHECK(cudaEventElapsedTime(&ms, ev[1], ev[3]));
                info->score_ms += ms;
                XSW_CHECK(cudaEventElapsedTime(&ms, ev[3], ev[4]));
                info->event_ms += ms;
                XSW_CHECK(cudaEventElapsedTime(&ms, ev[4], ev[5]));
                info->admit_ms += ms;
            }
        }
        waves = std::max(waves, w.waves);
    }
    if (info) {
        info->waves = waves;
        info->n_slots = per * n_pipes;
        info->walk_blocks_per_sm = walk_per_sm;
        info->launches = launches;
        info->walk_ms = walk;
    }
    if (std::getenv("XSCAT_TIMING")) {
        const auto t3 = std::chrono::steady_clock::now();
        auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
        std::fprintf(stderr, "[xscat] wave_run: prepare %.1f ms (memory %.1f, buffers %.1f, kernels %.1f), waves %.1f ms (%u waves), tail %.1f ms\n",
                     ms(host_t0, host_t1), ms(host_t0, host_ta), ms(host_ta, host_tb), ms(host_tb, host_t1),
                     ms(host_t1, host_t2), waves, ms(host_t2, t3));
    }
    return cudaSuccess;
}
#undef XSW_CHECK

cudaError_t wave_run(WaveEngine* e, const TransportParams& P, int sm_count, uint32_t n_slots, cudaStream_t s,
                     WaveInfo* info, cudaEvent_t start, int n_pipes)
{
    return wave_run_jobs(e, &P, 1, sm_count, n_slots, s, info, start, n_pipes);
}

} // namespace xsd
