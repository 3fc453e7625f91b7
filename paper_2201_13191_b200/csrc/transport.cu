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
#include "transport_core.cuh"

namespace xsd {

namespace {

constexpr int kWarps = 4; // warps per block
static_assert(32 * kWarps == kBlock, "mu-table stride");
#ifndef XSD_MIN_BLOCKS
#define XSD_MIN_BLOCKS 4
#endif

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

// Megakernel queue policy: a warp's slots and FIFOs in shared memory.
// Scoring task: pixel << 6 | slot (n_pixels < 2^26, checked on the host).
// The scoring FIFO has qlen = H * splitting + 1 entries and its tail wraps
// (atomicInc), so it can never fill; the free-path FIFO follows it.
struct WarpQ {
    static constexpr bool kBatchScores = false;
    Slot* slots;   // H slots, then the WarpHdr, then the FIFOs
    uint32_t hoff; // byte offset of the WarpHdr
    uint32_t qlen;
    __device__ __forceinline__ WarpHdr* hdr_() const
    {
        return reinterpret_cast<WarpHdr*>(reinterpret_cast<unsigned char*>(slots) + hoff);
    }
    __device__ __forceinline__ uint32_t* q_() const { return reinterpret_cast<uint32_t*>(hdr_() + 1); }
    __device__ __forceinline__ Slot& slot(int s) const { return slots[s]; }
    __device__ __forceinline__ uint32_t reserve_scores(int) const { return 0; }
    __device__ __forceinline__ void push_score(uint32_t, int s, uint32_t pixel) const
    {
        const uint32_t i = atomicInc(&hdr_()->tail, qlen - 1u);
        q_()[i] = pixel << 6 | (uint32_t)s;
    }
    __device__ __forceinline__ void push_free(int s) const
    {
        const uint32_t i = atomicAdd(&hdr_()->ftail, 1u);
        q_()[qlen + (i & (kFreeQ - 1))] = (uint32_t)s;
    }
    __device__ __forceinline__ void claim(int s) const { atomicAnd(&hdr_()->free_mask, ~(1ull << s)); }
    __device__ __forceinline__ void release(int s) const { atomicOr(&hdr_()->free_mask, 1ull << s); }
    __device__ __forceinline__ void fence() const { __threadfence_block(); }
    // statistics straight into the block's shared accumulators
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

} // namespace

// per-warp shared memory: slots, header, scoring + free-path FIFOs (8-aligned)
__host__ __device__ inline size_t warp_bytes_of(int H, int qlen)
{
    return ((size_t)H * sizeof(Slot) + sizeof(WarpHdr) + (size_t)(qlen + kFreeQ) * 4 + 15) & ~(size_t)15;
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
    // (slots are 16-byte aligned: Slot is read and written with 16-byte accesses)
    unsigned char* p = reinterpret_cast<unsigned char*>(sstart + P.n_bins + 1 + ((P.n_bins + 1) & 1));
    const size_t warp_bytes = warp_bytes_of(H, P.queue_len);
    unsigned char* wbase = p + (size_t)warp * warp_bytes;
    Slot* slots = reinterpret_cast<Slot*>(wbase);
    WarpHdr* hdr = reinterpret_cast<WarpHdr*>(wbase + (size_t)H * sizeof(Slot));
    uint32_t* q = reinterpret_cast<uint32_t*>(hdr + 1);
    const WarpQ qs{slots, (uint32_t)((size_t)H * sizeof(Slot)), qlen};
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
    uint32_t c_fp = 0, c_sc = 0, c_rays = 0, c_int = 0, c_iter = 0, c_wit = 0, c_uni = 0;

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
                history_start(P, B, qs, sstart, s, first + lane, st);
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
        w.ucells = 0;
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
            c_uni += w.ucells;
            const uint64_t var_base = (gwarp * H + tslot) * (uint64_t)P.var_cap;
            if (ttype == T_SCORE) { // REF run_history :178-193
                score_complete(P, B, qs, tslot, tpix, tpre, w.depth, var_base, st);
            } else {
                const bool hit = w.hit != 0;
                if (hit)
                    ++c_int;
                history_event<FMT>(P, B, qs, tslot, hit, hit ? hit_t(w) : 0.0, w.ix,
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
    sadd(B.diag + 7, c_uni);
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
static bool use_reg(const TransportParams& P) { return (P.G.fmt == kFmtP4 || P.G.fmt == kFmtP8) && P.n_pal <= 4; }

size_t transport_smem_bytes(const TransportParams& P)
{
    const size_t warp_bytes = warp_bytes_of(P.slots_per_warp, P.queue_len);
    const int n_tab = P.G.fmt == kFmtP4 ? P.n_pal : P.n_mats;
    return (size_t)(8 * P.n_bins + 32) * 8 + (size_t)(P.n_bins + 2) * 8 + kWarps * warp_bytes +
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
    if (P.G.fmt == kFmtP8) {
        if (use_reg(P))
            return skip ? transport_kernel<kFmtP8, true, true> : transport_kernel<kFmtP8, true, false>;
        return skip ? transport_kernel<kFmtP8, false, true> : transport_kernel<kFmtP8, false, false>;
    }
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
