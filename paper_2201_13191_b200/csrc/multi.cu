// multi.cu — the projector on several GPUs.
//
// A history is a pure function of (seed, angle, bin, photon) (REF rng.hpp:13-17,
// transport.cpp:122-123) and every tally is a fixed-point integer, so:
//  * one projection's history range splits into contiguous photon batches,
//    one per GPU (REF's chunk rule, transport.cpp:274-275, with one chunk per
//    GPU); the accumulators are summed (u64 adds) and finalized once, and the
//    image is bit-identical for any GPU count;
//  * scans split into contiguous angle ranges (REF run_scan's angle loop,
//    transport.cpp:405-420; the paper's projections across GPUs).
//
// Two ways to form the set of GPUs:
//  * multi-process (one process per GPU): xs_ctx_comm_init gives a context an
//    NCCL communicator.  Photon batches are combined by ncclReduce(ncclUint64,
//    ncclSum) into the root's accumulator; scan images are gathered to the
//    root with ncclSend / ncclRecv.  Before every collective the ranks agree on
//    success (an ncclAllReduce of the status), so a rank that failed makes all
//    ranks fail with its message instead of leaving the others waiting.
//  * one process (xs_group_*): one context per listed device, one host thread
//    per member.  The members' accumulators are read by the root's finalize
//    kernel directly over NVLink peer memory and summed as it dequantizes:
//    reduce and finalize are one pass, with no reduced copy written.  A device
//    may be listed more than once (members then share it; used by the tests on
//    one GPU).
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "capi_internal.h"
#include "host_common.h"

using xsh::Error;
using xsh::fail;

namespace {

void nccl_check(ncclResult_t r, const char* what)
{
    if (r != ncclSuccess)
        fail(XS_E_CUDA, "%s: NCCL error: %s", what, ncclGetErrorString(r));
}

template <typename T>
struct Dev {
    T* p = nullptr;
    size_t n = 0;
    void reserve(size_t count)
    {
        if (count <= n && p)
            return;
        if (p)
            cudaFree(p);
        p = nullptr;
        n = 0;
        xsi::cuda(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)), "cudaMalloc");
        n = count;
    }
    void release()
    {
        if (p)
            cudaFree(p);
        p = nullptr;
        n = 0;
    }
    ~Dev() { release(); }
};

// Communicator state of one context (xs_ctx_comm_init).
struct Comm {
    ncclComm_t comm = nullptr;
    int n = 1, rank = 0;
    Dev<int> flag;         // status agreement
    Dev<double> img[2];    // scan gather staging (primary, scatter)
    Dev<double> secs;
    ~Comm()
    {
        if (comm)
            ncclCommDestroy(comm);
    }
};

Comm* comm_of(xs_context* c)
{
    Comm* cm = static_cast<Comm*>(xsi::mgpu_slot(c));
    if (!cm)
        fail(XS_E_RUNTIME, "xscat-gpu: context has no communicator (xs_ctx_comm_init)");
    return cm;
}

// Runs f; then every rank learns whether any rank failed.  A rank that failed
// rethrows its own error; the others fail naming the first failing rank.
void agreed(xs_context* c, Comm* cm, const std::function<void()>& f)
{
    int bad = 0;
    Error err{0, std::string()};
    try {
        f();
    } catch (const Error& e) {
        err = e;
        bad = 1;
    }
    if (cm->n > 1) {
        // max over ranks of -(rank + 1) for the failing ranks: the lowest failing rank
        cudaStream_t s = xsi::stream(c);
        const int none = -(1 << 30);
        int v = bad ? -(cm->rank + 1) : none;
        cm->flag.reserve(1);
        xsi::cuda(cudaMemcpyAsync(cm->flag.p, &v, sizeof(int), cudaMemcpyHostToDevice, s), "H2D");
        nccl_check(ncclAllReduce(cm->flag.p, cm->flag.p, 1, ncclInt32, ncclMax, cm->comm, s), "ncclAllReduce");
        xsi::cuda(cudaMemcpyAsync(&v, cm->flag.p, sizeof(int), cudaMemcpyDeviceToHost, s), "D2H");
        xsi::cuda(cudaStreamSynchronize(s), "status agreement");
        if (v != none && !bad)
            fail(XS_E_RUNTIME, "xscat-gpu: rank %d failed", -v - 1);
    }
    if (bad)
        throw err;
}

} // namespace

namespace xsi {
void mgpu_release(xs_context* c)
{
    delete static_cast<Comm*>(mgpu_slot(c));
    mgpu_slot(c) = nullptr;
}
} // namespace xsi

// ============================================================ multi-process
extern "C" {

int xs_comm_unique_id(xs_comm_id* out)
{
    static_assert(sizeof(ncclUniqueId) <= sizeof(xs_comm_id), "xs_comm_id too small");
    try {
        ncclUniqueId id;
        nccl_check(ncclGetUniqueId(&id), "ncclGetUniqueId");
        std::memset(out, 0, sizeof *out);
        std::memcpy(out->internal, &id, sizeof id);
        return XS_OK;
    } catch (const Error& e) {
        return xsh::set_error(e.code, e.msg);
    }
}

int xs_ctx_comm_init(xs_context* c, int32_t n_ranks, int32_t rank, const xs_comm_id* id)
{
    return xsi::run(c, [&] {
        if (n_ranks < 1 || rank < 0 || rank >= n_ranks)
            fail(XS_E_OUT_OF_RANGE, "xs_ctx_comm_init: rank %d out of range (%d ranks)", rank, n_ranks);
        xsi::mgpu_release(c);
        auto cm = std::make_unique<Comm>();
        cm->n = n_ranks;
        cm->rank = rank;
        ncclUniqueId uid;
        std::memcpy(&uid, id->internal, sizeof uid);
        nccl_check(ncclCommInitRank(&cm->comm, n_ranks, uid, rank), "ncclCommInitRank");
        xsi::mgpu_slot(c) = cm.release();
    });
}

int xs_ctx_comm_size(const xs_context* c, int32_t* n_ranks, int32_t* rank)
{
    const Comm* cm = static_cast<const Comm*>(xsi::mgpu_slot(const_cast<xs_context*>(c)));
    *n_ranks = cm ? cm->n : 1;
    *rank = cm ? cm->rank : 0;
    return XS_OK;
}

int xs_simulate_scatter_stats_mgpu(xs_context* c, const xs_geometry* g, int32_t angle_idx, const xs_spectrum* spec,
                                   const xs_sim_config* cfg, int32_t root, xs_scatter_result* out, double* d_image)
{
    return xsi::run(c, [&] {
        Comm* cm = comm_of(c);
        if (root < 0 || root >= cm->n)
            fail(XS_E_OUT_OF_RANGE, "xs_simulate_scatter_stats_mgpu: root %d out of range", root);
        cudaStream_t s = xsi::stream(c);
        xs_accum_layout L{};
        uint64_t n = 0, h0 = 0, h1 = 0;
        unsigned long long* acc = nullptr;
        const auto t0 = std::chrono::steady_clock::now();
        agreed(c, cm, [&] {
            xsi::accumulate(c, *g, angle_idx, *spec, *cfg, 0, 0, nullptr); // REF's validation and messages
            n = xsi::history_count(*g, *spec, *cfg);
            L = xsi::layout(*g, *spec, *cfg);
            h0 = n * (uint64_t)cm->rank / (uint64_t)cm->n;
            h1 = n * (uint64_t)(cm->rank + 1) / (uint64_t)cm->n;
            acc = xsi::own_accum(c, L.words);
            xsi::cuda(cudaMemsetAsync(acc, 0, L.words * 8, s), "memset accum");
            xsi::accumulate(c, *g, angle_idx, *spec, *cfg, h0, h1, acc); // validates like REF
        });
        if (cm->n > 1) {
            const xsi::Range range("xscat: ncclReduce of the tallies");
            nccl_check(ncclReduce(acc, acc, L.words, ncclUint64, ncclSum, root, cm->comm, s), "ncclReduce");
        }
        const auto t1 = std::chrono::steady_clock::now();
        if (cm->rank == root) {
            const unsigned long long* src = acc;
            xsi::finalize(c, *g, *spec, *cfg, &src, 1, 0, n, out, d_image);
            if (std::getenv("XSCAT_TIMING")) {
                const auto t2 = std::chrono::steady_clock::now();
                std::fprintf(stderr, "[xscat] mgpu: accumulate %.1f ms, finalize %.1f ms\n",
                             std::chrono::duration<double, std::milli>(t1 - t0).count(),
                             std::chrono::duration<double, std::milli>(t2 - t1).count());
            }
        } else {
            xsi::cuda(cudaStreamSynchronize(s), "reduce");
            out->histories = h1 - h0;
        }
    });
}

int xs_run_scan_mgpu(xs_context* c, const xs_geometry* g, const xs_spectrum* spec, const xs_sim_config* cfg,
                     const int32_t* subset, int32_t n_subset, int32_t what, int32_t gather, int32_t root,
                     double* primary_out, double* scatter_out, double* seconds)
{
    return xsi::run(c, [&] {
        Comm* cm = comm_of(c);
        if (root < 0 || root >= cm->n)
            fail(XS_E_OUT_OF_RANGE, "xs_run_scan_mgpu: root %d out of range", root);
        cudaStream_t s = xsi::stream(c);
        agreed(c, cm, [&] { xsi::check_scan_args(g, cfg, subset, n_subset); });
        const bool want_p = what != 1, want_s = what != 0;
        const size_t np = (size_t)g->nu * g->nv;
        auto share = [&](int r, int& a0, int& a1) {
            a0 = (int)((int64_t)n_subset * r / cm->n);
            a1 = (int)((int64_t)n_subset * (r + 1) / cm->n);
        };
        int my0, my1;
        share(cm->rank, my0, my1);
        if (!gather || cm->n == 1) { // no exchange: this rank's range through xs_run_scan
            // (its D2H and host copies overlap the next angle's transport)
            if (my1 <= my0)
                return;
            const int st = xs_run_scan(c, g, spec, cfg, subset + my0, my1 - my0, what,
                                       primary_out ? primary_out + (size_t)my0 * np : nullptr,
                                       scatter_out ? scatter_out + (size_t)my0 * np : nullptr,
                                       seconds ? seconds + my0 : nullptr);
            if (st != XS_OK)
                fail(st, "%s", xs_last_error(c));
            return;
        }
        // rounds of up to kChunk angles per rank: compute on the device, copy this
        // rank's images out, then (gather) the root receives the round's images of
        // every other rank
        constexpr int kChunk = 16;
        int rounds = 0;
        for (int r = 0; r < cm->n; ++r) {
            int a0, a1;
            share(r, a0, a1);
            rounds = std::max(rounds, (a1 - a0 + kChunk - 1) / kChunk);
        }
        const bool do_gather = gather && cm->n > 1;
        const size_t stage = (size_t)kChunk * np * (do_gather && cm->rank == root ? (size_t)cm->n : 1);
        if (want_p)
            cm->img[0].reserve(stage);
        if (want_s)
            cm->img[1].reserve(stage);
        cm->secs.reserve((size_t)kChunk * cm->n);
        std::vector<double> sec_h((size_t)kChunk * cm->n, 0.0);
        for (int k = 0; k < rounds; ++k) {
            const int b0 = std::min(my1, my0 + k * kChunk), b1 = std::min(my1, b0 + kChunk);
            agreed(c, cm, [&] {
                if (b1 > b0) {
                    xsi::scan_device(c, g, spec, cfg, subset + b0, b1 - b0, what, want_p ? cm->img[0].p : nullptr,
                                     want_s ? cm->img[1].p : nullptr, sec_h.data());
                    for (int q = 0; q < 2; ++q) {
                        double* dst = q == 0 ? primary_out : scatter_out;
                        if (dst && (q == 0 ? want_p : want_s))
                            xsi::cuda(cudaMemcpyAsync(dst + (size_t)b0 * np, cm->img[q].p, (size_t)(b1 - b0) * np * 8,
                                                      cudaMemcpyDeviceToHost, s),
                                      "D2H");
                    }
                    if (seconds)
                        std::memcpy(seconds + b0, sec_h.data(), (size_t)(b1 - b0) * 8);
                    xsi::cuda(cudaMemcpyAsync(cm->secs.p, sec_h.data(), (size_t)(b1 - b0) * 8,
                                              cudaMemcpyHostToDevice, s),
                              "H2D");
                    xsi::cuda(cudaStreamSynchronize(s), "scan round");
                }
            });
            if (!do_gather)
                continue;
            const xsi::Range range("xscat: scan gather");
            nccl_check(ncclGroupStart(), "ncclGroupStart");
            for (int r = 0; r < cm->n; ++r) {
                int a0, a1;
                share(r, a0, a1);
                const int c0 = std::min(a1, a0 + k * kChunk), c1 = std::min(a1, c0 + kChunk);
                const size_t cnt = (size_t)(c1 - c0);
                if (r == root || cnt == 0)
                    continue;
                if (cm->rank == r) {
                    for (int q = 0; q < 2; ++q)
                        if (q == 0 ? want_p : want_s)
                            nccl_check(ncclSend(cm->img[q].p, cnt * np, ncclFloat64, root, cm->comm, s), "ncclSend");
                    nccl_check(ncclSend(cm->secs.p, cnt, ncclFloat64, root, cm->comm, s), "ncclSend");
                } else if (cm->rank == root) {
                    for (int q = 0; q < 2; ++q)
                        if (q == 0 ? want_p : want_s)
                            nccl_check(ncclRecv(cm->img[q].p + (size_t)r * kChunk * np, cnt * np, ncclFloat64, r,
                                                cm->comm, s),
                                       "ncclRecv");
                    nccl_check(ncclRecv(cm->secs.p + (size_t)r * kChunk, cnt, ncclFloat64, r, cm->comm, s),
                               "ncclRecv");
                }
            }
            nccl_check(ncclGroupEnd(), "ncclGroupEnd");
            if (cm->rank == root) {
                xsi::cuda(cudaMemcpyAsync(sec_h.data(), cm->secs.p, sec_h.size() * 8, cudaMemcpyDeviceToHost, s),
                          "D2H");
                for (int r = 0; r < cm->n; ++r) {
                    int a0, a1;
                    share(r, a0, a1);
                    const int c0 = std::min(a1, a0 + k * kChunk), c1 = std::min(a1, c0 + kChunk);
                    if (r == root || c1 <= c0)
                        continue;
                    for (int q = 0; q < 2; ++q) {
                        double* dst = q == 0 ? primary_out : scatter_out;
                        if (dst && (q == 0 ? want_p : want_s))
                            xsi::cuda(cudaMemcpyAsync(dst + (size_t)c0 * np, cm->img[q].p + (size_t)r * kChunk * np,
                                                      (size_t)(c1 - c0) * np * 8, cudaMemcpyDeviceToHost, s),
                                      "D2H");
                    }
                }
                xsi::cuda(cudaStreamSynchronize(s), "gather");
                for (int r = 0; r < cm->n; ++r) {
                    int a0, a1;
                    share(r, a0, a1);
                    const int c0 = std::min(a1, a0 + k * kChunk), c1 = std::min(a1, c0 + kChunk);
                    if (r != root && c1 > c0 && seconds)
                        std::memcpy(seconds + c0, sec_h.data() + (size_t)r * kChunk, (size_t)(c1 - c0) * 8);
                }
            } else {
                xsi::cuda(cudaStreamSynchronize(s), "gather");
            }
        }
    });
}

} // extern "C"

// ============================================================== one process
struct xs_group {
    std::vector<xs_context*> ctx;
    std::string err;
    bool peer_ok = true; // the root reads every member's memory directly
    std::vector<std::unique_ptr<Dev<unsigned long long>>> acc; // per member accumulator
    std::vector<std::unique_ptr<Dev<double>>> scan_buf[2];     // per member scan outputs (loop delegate)
    Dev<unsigned long long> staged;                            // members' accumulators copied to the root (no P2P)
};

namespace {

int group_run(xs_group* G, const std::function<void()>& f)
{
    try {
        xsi::cuda(cudaSetDevice(xsi::device(G->ctx[0])), "cudaSetDevice");
        f();
        G->err.clear();
        return XS_OK;
    } catch (const Error& e) {
        G->err = e.msg;
        return xsh::set_error(e.code, e.msg);
    } catch (const std::exception& e) {
        G->err = e.what();
        return xsh::set_error(XS_E_RUNTIME, e.what());
    }
}

// Runs f(i) for every member on its own host thread; the error of the lowest
// failing member wins (members hold increasing shares, so this is the error
// REF's sequential loop would have raised first).
void each_member(xs_group* G, const std::function<int(int)>& f)
{
    const int n = (int)G->ctx.size();
    std::vector<int> st(n, XS_OK);
    std::vector<std::string> msg(n);
    std::vector<std::thread> th;
    for (int i = 0; i < n; ++i)
        th.emplace_back([&, i] {
            st[i] = f(i);
            if (st[i] != XS_OK)
                msg[i] = xs_last_error(G->ctx[i]);
        });
    for (auto& t : th)
        t.join();
    for (int i = 0; i < n; ++i)
        if (st[i] != XS_OK)
            fail(st[i], "%s", msg[i].c_str());
}

void share(int64_t n, int parts, int i, int64_t& a0, int64_t& a1)
{
    a0 = n * i / parts;
    a1 = n * (i + 1) / parts;
}

} // namespace

extern "C" {

int xs_group_create(const int32_t* devices, int32_t n, xs_group** out)
{
    *out = nullptr;
    try {
        if (n < 1 || n > 16)
            fail(XS_E_OUT_OF_RANGE, "xs_group_create: 1..16 members supported (%d requested)", n);
        auto G = std::make_unique<xs_group>();
        for (int i = 0; i < n; ++i) {
            xs_context* c = nullptr;
            const int st = xs_ctx_create(devices[i], &c);
            if (st != XS_OK) {
                for (xs_context* x : G->ctx)
                    xs_ctx_destroy(x);
                fail(st, "%s", xs_last_error(nullptr));
            }
            G->ctx.push_back(c);
            G->acc.emplace_back(new Dev<unsigned long long>());
            G->scan_buf[0].emplace_back(new Dev<double>());
            G->scan_buf[1].emplace_back(new Dev<double>());
        }
        // the root reads the members' accumulators over NVLink
        const int root = devices[0];
        xsi::cuda(cudaSetDevice(root), "cudaSetDevice");
        for (int i = 1; i < n; ++i) {
            if (devices[i] == root)
                continue;
            int can = 0;
            xsi::cuda(cudaDeviceCanAccessPeer(&can, root, devices[i]), "cudaDeviceCanAccessPeer");
            if (!can) {
                G->peer_ok = false;
                continue;
            }
            const cudaError_t e = cudaDeviceEnablePeerAccess(devices[i], 0);
            if (e == cudaErrorPeerAccessAlreadyEnabled)
                cudaGetLastError();
            else
                xsi::cuda(e, "cudaDeviceEnablePeerAccess");
        }
        *out = G.release();
        return XS_OK;
    } catch (const Error& e) {
        return xsh::set_error(e.code, e.msg);
    }
}

void xs_group_destroy(xs_group* G)
{
    if (!G)
        return;
    for (size_t i = 0; i < G->ctx.size(); ++i) {
        cudaSetDevice(xsi::device(G->ctx[i]));
        G->acc[i].reset();
        G->scan_buf[0][i].reset();
        G->scan_buf[1][i].reset();
    }
    cudaSetDevice(xsi::device(G->ctx[0]));
    G->staged.release();
    for (xs_context* c : G->ctx)
        xs_ctx_destroy(c);
    delete G;
}

int32_t xs_group_size(const xs_group* G) { return G ? (int32_t)G->ctx.size() : 0; }

xs_context* xs_group_context(xs_group* G, int32_t i)
{
    return (G && i >= 0 && i < (int32_t)G->ctx.size()) ? G->ctx[i] : nullptr;
}

const char* xs_group_last_error(const xs_group* G) { return G ? G->err.c_str() : xsh::thread_error(); }

int xs_group_set_option(xs_group* G, const char* key, int64_t value)
{
    return group_run(G, [&] {
        for (xs_context* c : G->ctx)
            if (xs_ctx_set_option(c, key, value) != XS_OK)
                fail(XS_E_INVALID_ARGUMENT, "%s", xs_last_error(c));
    });
}

int xs_group_upload_phantom(xs_group* G, const xs_phantom* ph)
{
    return group_run(G, [&] {
        xs_context* root = G->ctx[0];
        const int st = xs_upload_phantom(root, ph);
        if (st != XS_OK)
            fail(st, "%s", xs_last_error(root));
        each_member(G, [&](int i) { return i == 0 ? XS_OK : xs_ctx_copy_scene(G->ctx[i], root); });
    });
}

int xs_group_upload_response(xs_group* G, const xs_response* r)
{
    return group_run(G, [&] {
        for (xs_context* c : G->ctx) {
            const int st = xs_upload_response(c, r);
            if (st != XS_OK)
                fail(st, "%s", xs_last_error(c));
        }
    });
}

int xs_group_simulate_scatter_stats(xs_group* G, const xs_geometry* g, int32_t angle_idx, const xs_spectrum* spec,
                                    const xs_sim_config* cfg, xs_scatter_result* out)
{
    return group_run(G, [&] {
        const int n = (int)G->ctx.size();
        xs_context* root = G->ctx[0];
        // REF's validation and messages first (the root's view of the call)
        const int vst = xsi::run(root, [&] { xsi::accumulate(root, *g, angle_idx, *spec, *cfg, 0, 0, nullptr); });
        if (vst != XS_OK)
            fail(vst, "%s", xs_last_error(root));
        const uint64_t nh = xsi::history_count(*g, *spec, *cfg);
        const xs_accum_layout L = xsi::layout(*g, *spec, *cfg);
        each_member(G, [&](int i) {
            xs_context* c = G->ctx[i];
            return xsi::run(c, [&] {
                int64_t a0, a1;
                share((int64_t)nh, n, i, a0, a1);
                G->acc[i]->reserve(L.words);
                xsi::cuda(cudaMemsetAsync(G->acc[i]->p, 0, L.words * 8, xsi::stream(c)), "memset accum");
                xsi::accumulate(c, *g, angle_idx, *spec, *cfg, (uint64_t)a0, (uint64_t)a1, G->acc[i]->p);
                xsi::cuda(cudaStreamSynchronize(xsi::stream(c)), "member transport");
            });
        });
        std::vector<const unsigned long long*> srcs(n);
        for (int i = 0; i < n; ++i)
            srcs[i] = G->acc[i]->p;
        if (!G->peer_ok) { // no P2P path: copy the members' accumulators to the root first
            G->staged.reserve(L.words * (size_t)n);
            for (int i = 1; i < n; ++i) {
                xsi::cuda(cudaMemcpyPeer(G->staged.p + (size_t)i * L.words, xsi::device(root), G->acc[i]->p,
                                         xsi::device(G->ctx[i]), L.words * 8),
                          "cudaMemcpyPeer");
                srcs[i] = G->staged.p + (size_t)i * L.words;
            }
        }
        const int st = xsi::run(root, [&] { xsi::finalize(root, *g, *spec, *cfg, srcs.data(), n, 0, nh, out, nullptr); });
        if (st != XS_OK)
            fail(st, "%s", xs_last_error(root));
    });
}

int xs_group_run_scan(xs_group* G, const xs_geometry* g, const xs_spectrum* spec, const xs_sim_config* cfg,
                      const int32_t* subset, int32_t n_subset, int32_t what, double* primary_out,
                      double* scatter_out, double* seconds)
{
    return group_run(G, [&] {
        xsi::check_scan_args(g, cfg, subset, n_subset);
        const int n = (int)G->ctx.size();
        const size_t np = (size_t)g->nu * g->nv;
        each_member(G, [&](int i) {
            int64_t a0, a1;
            share(n_subset, n, i, a0, a1);
            if (a1 <= a0)
                return (int)XS_OK;
            return xs_run_scan(G->ctx[i], g, spec, cfg, subset + a0, (int32_t)(a1 - a0), what,
                               primary_out ? primary_out + (size_t)a0 * np : nullptr,
                               scatter_out ? scatter_out + (size_t)a0 * np : nullptr,
                               seconds ? seconds + a0 : nullptr);
        });
    });
}

int xs_group_run_iterative_correction(xs_group* G, const double* raw_intensity, const double* flatfield,
                                      const xs_geometry* g, const xs_spectrum* spec, const xs_correction_config* cfg,
                                      int32_t n_materials, const xs_material* materials, float* corrected_volume,
                                      double* corrected_stack, xs_iteration_report* reports, int32_t device_ptrs)
{
    return group_run(G, [&] {
        xs_context* root = G->ctx[0];
        const int n = (int)G->ctx.size();
        // the loop's scatter and primary scans, sharded by angle: the members get
        // the current (segmented) scene device to device, scan their angle range
        // into their own buffers, and the images come back into the root's stack
        xsi::set_scan_hook(root, [G, root, n](const xs_geometry* gm, const xs_spectrum* sp, const xs_sim_config* sc,
                                              const int32_t* subset, int32_t n_sub, int32_t what, double* d_primary,
                                              double* d_scatter) {
            const size_t np = (size_t)gm->nu * gm->nv;
            each_member(G, [&](int i) {
                int64_t a0, a1;
                share(n_sub, n, i, a0, a1);
                xs_context* c = G->ctx[i];
                if (a1 <= a0)
                    return (int)XS_OK;
                return xsi::run(c, [&] {
                    if (i > 0) {
                        const int st = xs_ctx_copy_scene(c, root);
                        if (st != XS_OK)
                            fail(st, "%s", xs_last_error(c));
                    }
                    const size_t cnt = (size_t)(a1 - a0) * np;
                    double* dp = nullptr;
                    double* ds = nullptr;
                    if (i == 0) {
                        dp = d_primary ? d_primary + (size_t)a0 * np : nullptr;
                        ds = d_scatter ? d_scatter + (size_t)a0 * np : nullptr;
                    } else {
                        if (d_primary) {
                            G->scan_buf[0][i]->reserve(cnt);
                            dp = G->scan_buf[0][i]->p;
                        }
                        if (d_scatter) {
                            G->scan_buf[1][i]->reserve(cnt);
                            ds = G->scan_buf[1][i]->p;
                        }
                    }
                    xsi::scan_device(c, gm, sp, sc, subset + a0, (int32_t)(a1 - a0), what, dp, ds, nullptr);
                    if (i > 0) {
                        cudaStream_t s = xsi::stream(c);
                        if (d_primary)
                            xsi::cuda(cudaMemcpyPeerAsync(d_primary + (size_t)a0 * np, xsi::device(root), dp,
                                                          xsi::device(c), cnt * 8, s),
                                      "cudaMemcpyPeerAsync");
                        if (d_scatter)
                            xsi::cuda(cudaMemcpyPeerAsync(d_scatter + (size_t)a0 * np, xsi::device(root), ds,
                                                          xsi::device(c), cnt * 8, s),
                                      "cudaMemcpyPeerAsync");
                        xsi::cuda(cudaStreamSynchronize(s), "scan gather");
                    }
                });
            });
        });
        const int st = xs_run_iterative_correction(root, raw_intensity, flatfield, g, spec, cfg, n_materials,
                                                   materials, corrected_volume, corrected_stack, reports,
                                                   device_ptrs);
        xsi::set_scan_hook(root, nullptr);
        if (st != XS_OK)
            fail(st, "%s", xs_last_error(root));
    });
}

} // extern "C"
