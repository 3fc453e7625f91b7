// capi.cu — the extern "C" boundary of libxscatgpu.so (include/xscat_gpu.h).
//
// Owns a per-device context (stream, device buffers, uploaded scene), the
// re-encoding of the phantom into the device voxel format, kernel launches,
// and the mapping of device error records to REF's exception types/messages.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <functional>
#include <string>
#include <thread>
#include <vector>

#include "capi_internal.h"
#include "host_common.h"
#include "xs_types.h"

namespace xsd {
size_t transport_smem_bytes(const TransportParams& P);
int transport_block_size();
int transport_pick_slots(TransportParams& P, int max_slots, size_t budget);
cudaError_t transport_prepare(const TransportParams& P, size_t smem, int* blocks_per_sm);
cudaError_t launch_transport(const TransportParams& P, int grid, size_t smem, cudaStream_t s);
cudaError_t launch_primary(const PrimaryParams& P, cudaStream_t s);
size_t levels_scratch_bytes(const Grid& G, const int* edges, int n_levels);
size_t correct_stats_bytes(int n_views);
size_t fbp_filter_smem(int nu);
cudaError_t launch_fbp_filter(const double* in, double* out, const double* kern, int nu, int nv, int n_views,
                              double R, double du, double dv, cudaStream_t s);
cudaError_t launch_fbp_backproject(const double* q, const void* views, int n_views, int nu, int nv,
                                   const int dims[3], const double voxel[3], double R, double du, double dv,
                                   float* vol, cudaStream_t s);
cudaError_t launch_i2a(const double* in, const double* flat, double* out, size_t npix, int n_img, void* stats,
                       int sm_count, cudaStream_t s);
cudaError_t launch_correct(const double* a, const double* ip, const double* is, double* out, size_t n, void* stats,
                           int sm_count, cudaStream_t s);
cudaError_t launch_correction_tail(const double* primary, const double* scatter, const double* a, double* tmp,
                                   double* out, int nu, int nv, int n_views, int nu_out, int nv_out, void* stats,
                                   cudaStream_t s);
cudaError_t launch_walk_probe(const TransportParams& P, unsigned long long* iters, cudaStream_t s);
cudaError_t launch_mark_levels(uint8_t* vox, const Grid& G, int fmt, const int* edges, int n_levels,
                               void* scratch, int sm_count, cudaStream_t s);
cudaError_t launch_run_field(uint8_t* vox, const Grid& G, int axis, int sign, int shift, int cap, int sm_count,
                             cudaStream_t s);
size_t seg_ctl_bytes();
size_t otsu_scratch_bytes(int bins, int n_classes);
cudaError_t launch_seg_reset(void* ctl, cudaStream_t s);
cudaError_t launch_otsu(const float* vol, const int dims[3], int n_classes, int bins, void* ctl, void* scratch,
                        double* thr, int sm_count, cudaStream_t s);
cudaError_t launch_segment_labels(const float* vol, uint64_t n, const double* thr, int n_thr, uint8_t* labels,
                                  int sm_count, cudaStream_t s);
cudaError_t launch_density_phantom(const uint8_t* labels, const float* vol, const int src[3], const int tgt[3],
                                   const int* cls_mat, const double* cls_dens, int n_labels, const double* thr,
                                   int n_thr, uint8_t* id_out, float* dens_out, void* ctl, int sm_count,
                                   cudaStream_t s);
cudaError_t launch_phantom_scan(const uint8_t* ids, const float* dens, uint64_t n, int n_materials,
                                uint32_t has_tables, void* ctl, int sm_count, cudaStream_t s);
cudaError_t launch_phantom_encode(const uint8_t* ids, const float* dens, const unsigned long long* pal, int n_pal,
                                  const Grid& G, int fmt, uint8_t* vox, float* vdens, int sm_count, cudaStream_t s);
size_t ncc_scratch_bytes();
cudaError_t launch_ncc(const float* x1, const float* x2, uint64_t n, void* scratch, cudaStream_t s);
struct WaveEngine;
WaveEngine* wave_create();
void wave_destroy(WaveEngine* e);
cudaError_t wave_run(WaveEngine* e, const TransportParams& P, int sm_count, uint32_t n_slots, cudaStream_t s,
                     WaveInfo* info, cudaEvent_t start, int n_pipes);
cudaError_t wave_run_jobs(WaveEngine* e, const TransportParams* jobs, int n_jobs, int sm_count, uint32_t n_slots,
                          cudaStream_t s, WaveInfo* info, cudaEvent_t start, int n_pipes);
cudaError_t launch_finalize_image(const unsigned long long* const* srcs, int n_src, uint64_t off_image,
                                  uint64_t off_var, uint64_t npix, int log2_img, double n_hist, int track_var,
                                  double* image, double* var, cudaStream_t s);
cudaError_t launch_sg(const double* in, double* tmp, double* out, int nu, int nv, int n_images,
                      int half, const double* K, cudaStream_t s);
cudaError_t launch_interp(const double* in, double* out, const InterpEntry* tab, int n_tgt,
                          size_t npix, cudaStream_t s);
cudaError_t launch_upsample(const double* in, double* tmp, double* out, int nu, int nv,
                            int n_images, int nu_out, int nv_out, cudaStream_t s);
cudaError_t launch_downsample(const double* in, double* out, int nu, int nv, int n_images,
                              int nu_out, int nv_out, cudaStream_t s);
} // namespace xsd

using xsh::Error;
using xsh::fail;

namespace {

constexpr double kPi = 3.14159265358979323846;

void cuda_check(cudaError_t e, const char* what)
{
    if (e != cudaSuccess)
        fail(XS_E_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

// Growable device buffer.
template <typename T>
struct DevBuf {
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
        cuda_check(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)), "cudaMalloc");
        n = count;
    }
    void release()
    {
        if (p)
            cudaFree(p);
        p = nullptr;
        n = 0;
    }
};

// Growable pinned host buffer (H2D staging).
template <typename T>
struct PinBuf {
    T* p = nullptr;
    size_t n = 0;
    void reserve(size_t count)
    {
        if (count <= n && p)
            return;
        if (p)
            cudaFreeHost(p);
        p = nullptr;
        n = 0;
        cuda_check(cudaMallocHost(&p, std::max<size_t>(count, 1) * sizeof(T)), "cudaMallocHost");
        n = count;
    }
    void release()
    {
        if (p)
            cudaFreeHost(p);
        p = nullptr;
        n = 0;
    }
};

// Host copy of a table (the C-ABI inputs are borrowed pointers).
struct HTab {
    std::vector<double> x, y;
    xs_table view() const { return xs_table{static_cast<int32_t>(x.size()), x.data(), y.data()}; }
    void set(const xs_table& t)
    {
        x.assign(t.x, t.x + std::max(t.n, 0));
        y.assign(t.y, t.y + std::max(t.n, 0));
    }
};

struct HMat {
    std::string name;
    double z_eff = 0, density_ref = 0;
    HTab t[6];
    xs_material view() const
    {
        xs_material m;
        m.name = name.c_str();
        m.z_eff = z_eff;
        m.density_ref = density_ref;
        m.mu = t[0].view();
        m.sigma_incoh = t[1].view();
        m.sigma_coh = t[2].view();
        m.sigma_pe = t[3].view();
        m.s_factor = t[4].view();
        m.f_factor = t[5].view();
        return m;
    }
};

} // namespace

struct xs_context {
    int device = 0;
    int sm_count = 148;
    cudaStream_t own = nullptr, stream = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    std::string err;

    // scene
    bool have_phantom = false, have_response = false;
    xsd::Grid grid{};
    int n_mats = 0;
    std::vector<HMat> mats;
    HTab resp_dqe, resp_dep;
    xsd::MatDesc mat_desc[xsd::kMaxMaterials]{};
    xsd::TabDesc resp_desc{};
    int n_pal = 0;
    uint8_t pal_mat[xsd::kMaxPalette]{};
    float pal_dens[xsd::kMaxPalette]{};
    DevBuf<uint8_t> vox;
    DevBuf<float> dens;
    DevBuf<double> tabs;
    PinBuf<uint8_t> pin_vox;
    PinBuf<uint8_t> pin_raw;  // staging of the raw id / density arrays (device-encoded upload)
    int upload_path = 1;      // 0: host encode + H2D of the grid; 1: H2D of the raw arrays + device encode
    PinBuf<float> pin_dens;
    uint64_t last_upload_bytes = 0;

    // scratch
    DevBuf<unsigned long long> accum;
    DevBuf<uint64_t> bin_start, bin_count;
    DevBuf<double> bin_e, bin_w, prim_atten, prim_w, prim_resp;
    DevBuf<unsigned long long> pool;
    DevBuf<xsd::DevStatus> status;
    DevBuf<uint32_t> var_pix;
    DevBuf<double> var_val;
    DevBuf<double> img, var, pp_a, pp_b, pp_c, pp_k;
    DevBuf<xsd::InterpEntry> interp_tab;
    DevBuf<uint8_t> lvl_scratch;
    DevBuf<double> scan_img[2]; // run_scan: double-buffered scatter images ...
    PinBuf<double> scan_pin[2]; // ... and their pinned staging
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t scan_ev[2] = {nullptr, nullptr}, scan_done[2] = {nullptr, nullptr};
    cudaEvent_t up_done[4] = {nullptr, nullptr, nullptr, nullptr}; // staged phantom upload ring
    DevBuf<double> cc_in[3], cc_out, cc_tmp, cc_sg, cc_full;
    DevBuf<unsigned long long> cc_stats;
    DevBuf<double> fbp_in, fbp_q, fbp_k, fbp_views;
    DevBuf<float> fbp_vol;
    DevBuf<unsigned char> seg_ctl, seg_scratch; // segmentation stage (segment.cu)
    DevBuf<double> seg_thr;
    DevBuf<uint8_t> seg_ids, seg_labels;
    DevBuf<float> seg_dens, seg_vol;
    DevBuf<unsigned long long> seg_pal;
    DevBuf<double> loop_a, loop_c, loop_scat, loop_prim, loop_flat, loop_ncc; // iterative correction
    DevBuf<float> loop_vol[2];
    int smem_kb = 48; // per transport block: 4 blocks/SM leave 60 KB of L1
    int max_slots = 64;
    int macro_skip = 2;  // 0: voxel walk, 1: cross uniform blocks, 2: decided per phantom at upload
    bool skip_pays = true; // walk probe of the uploaded phantom (launch_walk_probe)
    DevBuf<unsigned long long> probe;

    xs_launch_stats last{};
    int grab = 64;
    int engine = 1;                  // 0: megakernel (transport.cu), 1: wavefront (wavefront.cu)
    std::vector<int> lvl_edges2{2, 8, 32}; // uniform-block edges with two level bits (C3 sweeps)
    int lvl_edge1 = 8;                      // ... with one level bit
    std::vector<int> lvl_edges3{2, 4, 8, 16, 32, 64, 128}; // ... with three (8-bit palette; edge 2 = 2^3 sub-blocks of mixed bricks)
    bool compact_palette = false;           // 4-bit palette for <= 8 pairs (half the bytes, fewer level bits)
    bool runs = true;                       // run field in the spare P8 bits (Grid::run_*)
    int run_bits = 0;                       // of the uploaded grid
    int run_key = -1;                       // axis * 2 + (sign > 0) the field holds; -1: none
    uint32_t wave_slots = 1u << 24;  // live histories of the wavefront engine (2^20 -> 2^22: +6% on C3; 2^23, 2^24: -1% each)
    int wave_pipes = 2;              // concurrent wavefront pipelines (streams)
    xsd::WaveEngine* wave = nullptr;
    // device scans: up to scan_jobs consecutive angles in one engine run, a
    // drained pipeline taking the next angle (scan_group); 1 = angle by angle
    static constexpr int kMaxScanJobs = 32;
    int scan_jobs = 8;
    DevBuf<unsigned long long> job_accum[kMaxScanJobs];
    DevBuf<double> job_img; // images of a group whose caller keeps none

    // multi-GPU (multi.cu): the NCCL communicator of xs_ctx_comm_init, and
    // the scan delegate a group installs on its root so the correction
    // loop's scans are sharded by angle over the group's devices
    void* mgpu = nullptr;
    xsi::ScanHook scan_hook;
};

namespace {

// --------------------------------------------------------------- plumbing
template <typename F>
int guard(xs_context* ctx, F&& f)
{
    try {
        if (ctx)
            cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
        f();
        return XS_OK;
    } catch (const Error& e) {
        if (ctx)
            ctx->err = e.msg;
        return xsh::set_error(e.code, e.msg);
    } catch (const std::exception& e) {
        if (ctx)
            ctx->err = e.what();
        return xsh::set_error(XS_E_RUNTIME, e.what());
    }
}

void rebuild_tables(xs_context* c)
{
    std::vector<double> buf;
    std::vector<xs_material> views(c->mats.size());
    for (size_t i = 0; i < c->mats.size(); ++i)
        views[i] = c->mats[i].view();
    if (!views.empty())
        xsh::pack_materials(views.data(), static_cast<int>(views.size()), buf, c->mat_desc);
    if (c->have_response)
        c->resp_desc = xsh::pack_table(c->resp_dep.view(), buf);
    if (buf.empty())
        buf.push_back(0.0);
    c->tabs.reserve(buf.size());
    cuda_check(cudaMemcpyAsync(c->tabs.p, buf.data(), buf.size() * sizeof(double),
                               cudaMemcpyHostToDevice, c->stream),
               "upload tables");
    cuda_check(cudaStreamSynchronize(c->stream), "upload tables");
}

void require_scene(const xs_context* c)
{
    if (!c->have_phantom)
        fail(XS_E_RUNTIME, "xscat-gpu: no phantom uploaded (xs_upload_phantom)");
    if (!c->have_response)
        fail(XS_E_RUNTIME, "xscat-gpu: no detector response uploaded (xs_upload_response)");
}

void check_angle(const xs_geometry& g, int angle_idx, const char* who)
{
    if (angle_idx < 0 || angle_idx >= g.n_angles)
        fail(XS_E_OUT_OF_RANGE, "%s: angle index out of range", who);
}

// Maps the device error record onto REF's exception type + message.
void check_status(xs_context* c, int angle_idx, const xs_spectrum* spec)
{
    xsd::DevStatus s;
    cuda_check(cudaMemcpyAsync(&s, c->status.p, sizeof s, cudaMemcpyDeviceToHost, c->stream),
               "status readback");
    cuda_check(cudaStreamSynchronize(c->stream), "kernel execution");
    if (s.code == 0)
        return;
    const double e = s.energy;
    switch (s.what) {
    case xsd::kErrNonFinite:
        fail(XS_E_RUNTIME,
             "simulate_scatter: non-finite contribution (angle %d, bin %d, E %f keV) - physics "
             "tables corrupt?",
             angle_idx, s.bin, e);
    case xsd::kErrTableRange:
        fail(XS_E_OUT_OF_RANGE, "table: query %f outside the tabulated range", e);
    case xsd::kErrTallyOverflow:
        fail(XS_E_RUNTIME, "simulate_scatter: fixed-point tally overflow (value %g)", s.value);
    case xsd::kErrSigmaIncoh:
        fail(XS_E_RUNTIME, "p_lambda_compton: vanishing incoherent cross section at %f keV", e);
    case xsd::kErrSigmaCoh:
        fail(XS_E_RUNTIME, "p_lambda_rayleigh: vanishing coherent cross section at %f keV", e);
    case xsd::kErrSigmaAll: {
        const int m = static_cast<int>(s.value);
        fail(XS_E_RUNTIME, "select_interaction: all cross sections vanish at %f keV in %s", e,
             (m >= 0 && m < (int)c->mats.size()) ? c->mats[m].name.c_str() : "?");
    }
    case xsd::kErrComptonS:
        fail(XS_E_RUNTIME, "sample_compton: S vanishes over the kinematic range at %f keV", e);
    case xsd::kErrStuck:
        fail(XS_E_RUNTIME, "simulate_scatter: transport did not terminate (E %f keV, site %g) - corrupt state", e, s.value);
    case xsd::kErrRayleighF:
        fail(XS_E_RUNTIME, "sample_rayleigh: F vanishes over the kinematic range at %f keV", e);
    default:
        if (s.code == XS_E_INVALID_ARGUMENT)
            fail(XS_E_INVALID_ARGUMENT, "trace: non-finite ray");
        fail(s.code, "device error %d", s.what);
    }
    (void)spec;
}

// ------------------------------------------------------ phantom encoding
struct PairKey {
    uint8_t id;
    uint32_t dens_bits;
    bool operator==(const PairKey& o) const { return id == o.id && dens_bits == o.dens_bits; }
    bool operator<(const PairKey& o) const
    {
        return id != o.id ? id < o.id : dens_bits < o.dens_bits;
    }
};

struct ScanResult {
    size_t first_bad = SIZE_MAX;
    int bad_code = 0;
    std::string bad_msg;
    std::vector<PairKey> pairs; // up to 257 distinct
};

// REF validate_phantom's per-voxel checks (phantom.cpp:42-54), in its order;
// empty when the voxel is valid.
std::string voxel_error(const xs_phantom& ph, const std::vector<int>& has_tables, uint8_t id, float d)
{
    if (id >= ph.n_materials)
        return "phantom: material id " + std::to_string(id) + " has no loaded material";
    if (id != 0 && !has_tables[id])
        return "phantom: material id " + std::to_string(id) + " (" +
               std::string(ph.materials[id].name ? ph.materials[id].name : "?") + ") has no tables";
    if (!(d >= 0.0f))
        return "phantom: negative density";
    if (id == 0 && d != 0.0f)
        return "phantom: vacuum voxel with nonzero density";
    return std::string();
}

// REF validate_phantom (phantom.cpp:33-56) fused with palette discovery.
void scan_phantom(const xs_phantom& ph, const std::vector<int>& has_tables, ScanResult& out)
{
    const size_t n = (size_t)ph.dims[0] * ph.dims[1] * ph.dims[2];
    const unsigned nt = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
    std::vector<ScanResult> part(nt);
    std::vector<std::thread> th;
    for (unsigned t = 0; t < nt; ++t)
        th.emplace_back([&, t] {
            ScanResult& r = part[t];
            const size_t b = n * t / nt, e = n * (t + 1) / nt;
            PairKey last{255, 0xFFFFFFFFu};
            bool have_last = false;
            for (size_t i = b; i < e; ++i) {
                const uint8_t id = ph.material_id[i];
                const float d = ph.density[i];
                uint32_t bits;
                std::memcpy(&bits, &d, 4);
                if (have_last && last.id == id && last.dens_bits == bits)
                    continue;
                if (id >= ph.n_materials) {
                    r.first_bad = i;
                    r.bad_code = 1;
                    r.bad_msg = "phantom: material id " + std::to_string(id) + " has no loaded material";
                    return;
                }
                if (id != 0 && !has_tables[id]) {
                    r.first_bad = i;
                    r.bad_msg = "phantom: material id " + std::to_string(id) + " (" +
                                std::string(ph.materials[id].name ? ph.materials[id].name : "?") +
                                ") has no tables";
                    return;
                }
                if (!(d >= 0.0f)) {
                    r.first_bad = i;
                    r.bad_msg = "phantom: negative density";
                    return;
                }
                if (id == 0 && d != 0.0f) {
                    r.first_bad = i;
                    r.bad_msg = "phantom: vacuum voxel with nonzero density";
                    return;
                }
                const PairKey k{id, bits};
                last = k;
                have_last = true;
                if (r.pairs.size() <= (size_t)xsd::kMaxPalette &&
                    std::find(r.pairs.begin(), r.pairs.end(), k) == r.pairs.end())
                    r.pairs.push_back(k);
            }
        });
    for (auto& t : th)
        t.join();
    for (auto& r : part) {
        if (r.first_bad < out.first_bad) {
            out.first_bad = r.first_bad;
            out.bad_msg = r.bad_msg;
        }
        for (const auto& k : r.pairs)
            if (out.pairs.size() <= (size_t)xsd::kMaxPalette &&
                std::find(out.pairs.begin(), out.pairs.end(), k) == out.pairs.end())
                out.pairs.push_back(k);
    }
    std::sort(out.pairs.begin(), out.pairs.end());
}

// Re-encodes the x-fastest grid into 4x4x4 bricks (P4 nibbles / P8 bytes /
// raw id + density), parallel over brick layers.
// vox / dens are (pinned) staging buffers of encoded_bytes(); every byte is written.
void encode_phantom(const xs_phantom& ph, int fmt, const std::vector<PairKey>& pal, uint8_t* vox,
                    float* dens, int nbx, int nby, int nbz)
{
    const int nx = ph.dims[0], ny = ph.dims[1], nz = ph.dims[2];
    const size_t layer_bytes = (size_t)nbx * nby * (fmt == xsd::kFmtP4 ? 32 : 64);
    const unsigned nt = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
    std::atomic<int> next{0};
    std::vector<std::thread> th;
    for (unsigned t = 0; t < nt; ++t)
        th.emplace_back([&] {
            for (;;) {
                const int bz = next.fetch_add(1);
                if (bz >= nbz)
                    return;
                std::memset(vox + (size_t)bz * layer_bytes, 0, layer_bytes); // padding voxels = code 0
                if (fmt == xsd::kFmtRaw)
                    std::memset(dens + (size_t)bz * nbx * nby * 64, 0, (size_t)nbx * nby * 64 * 4);
                PairKey last{255, 0xFFFFFFFFu};
                int last_code = 0;
                for (int z = bz * 4; z < std::min(nz, bz * 4 + 4); ++z)
                    for (int y = 0; y < ny; ++y)
                        for (int x = 0; x < nx; ++x) {
                            const size_t src = (size_t)x + (size_t)nx * ((size_t)y + (size_t)ny * z);
                            const size_t brick =
                                (size_t)(x >> 2) + (size_t)nbx * ((size_t)(y >> 2) + (size_t)nby * (z >> 2));
                            const size_t cell =
                                (brick << 6) | (size_t)((x & 3) | ((y & 3) << 2) | ((z & 3) << 4));
                            const uint8_t id = ph.material_id[src];
                            if (fmt == xsd::kFmtRaw) {
                                vox[cell] = id;
                                dens[cell] = ph.density[src];
                                continue;
                            }
                            uint32_t bits;
                            std::memcpy(&bits, &ph.density[src], 4);
                            int code = last_code;
                            if (!(last.id == id && last.dens_bits == bits)) {
                                const PairKey k{id, bits};
                                code = (int)(std::lower_bound(pal.begin(), pal.end(), k) - pal.begin());
                                last = k;
                                last_code = code;
                            }
                            if (fmt == xsd::kFmtP4)
                                vox[cell >> 1] |= (uint8_t)(code << ((cell & 1) * 4));
                            else
                                vox[cell] = (uint8_t)code;
                        }
            }
        });
    for (auto& t : th)
        t.join();
}

// Host view of the device SegCtl record (segment.cu): first_bad at byte 8,
// n_pairs / overflow at 16 / 20, the pair set at 56.
struct SegCtlView {
    const unsigned char* p;
    explicit SegCtlView(const unsigned char* b) : p(b) {}
    template <typename T>
    T at(size_t off) const
    {
        T v;
        std::memcpy(&v, p + off, sizeof v);
        return v;
    }
    unsigned long long first_bad() const { return at<unsigned long long>(8); }
    uint32_t n_pairs() const { return at<uint32_t>(16); }
    uint32_t overflow() const { return at<uint32_t>(20); }
    int32_t status() const { return at<int32_t>(24); }
    // distinct pairs, sorted; more than kMaxPalette entries = the raw format
    void pairs(std::vector<PairKey>& out) const
    {
        out.clear();
        if (overflow() || n_pairs() > (uint32_t)xsd::kMaxPalette) {
            out.resize(xsd::kMaxPalette + 1);
            return;
        }
        for (int i = 0; i < 1024; ++i) {
            const unsigned long long k = at<unsigned long long>(56 + 8 * (size_t)i);
            if (k != ~0ull)
                out.push_back(PairKey{(uint8_t)(k >> 32), (uint32_t)k});
        }
        std::sort(out.begin(), out.end());
    }
};

// --------------------------------------------------------- scatter launch
struct Plan {
    std::vector<uint64_t> counts, start;
    xs_accum_units units;
    xs_accum_layout layout;
    uint64_t n_hist;
};

Plan make_plan(const xs_geometry& g, const xs_spectrum& spec, const xs_sim_config& cfg)
{
    Plan p;
    if (spec.n_bins > xsd::kMaxBins)
        fail(XS_E_UNSUPPORTED, "xscat-gpu: at most %d spectrum bins supported", xsd::kMaxBins);
    p.counts = xsh::apportion(spec, cfg.photons_total);
    p.start.resize(spec.n_bins + 1);
    p.start[0] = 0;
    for (int b = 0; b < spec.n_bins; ++b)
        p.start[b + 1] = p.start[b] + p.counts[b];
    p.n_hist = p.start[spec.n_bins];
    p.units = xs_accum_units_make(&g, &spec, p.counts.data());
    p.layout = xs_accum_layout_make(g.nu, g.nv, spec.n_bins, cfg.track_variance);
    return p;
}

void validate_call(const xs_geometry& g, int angle, const xs_spectrum& spec,
                   const xs_sim_config& cfg, const char* who)
{
    xsh::validate_sim_config(cfg);
    xsh::validate_spectrum(spec);
    xsh::validate_geometry(g);
    check_angle(g, angle, who);
}

// The run field (Grid::run_*) for this projection's travel direction,
// source -> detector: the dominant in-plane axis and its sign.  Rewritten
// only when that changes (four times per full circle).
// the run field's key (axis * 2 + sign) for a projection: angles with equal
// keys share the field and can run in one engine call
int run_key_of(const xsh::Frame& f)
{
    const double dx = f.center[0] - f.src[0], dy = f.center[1] - f.src[1];
    const int axis = std::fabs(dx) >= std::fabs(dy) ? 0 : 1;
    const int sign = (axis == 0 ? dx : dy) > 0.0 ? 1 : -1;
    return axis * 2 + (sign > 0 ? 1 : 0);
}

void ensure_runs(xs_context* c, const xsh::Frame& f)
{
    if (!c->run_bits)
        return;
    const double dx = f.center[0] - f.src[0], dy = f.center[1] - f.src[1];
    const int axis = std::fabs(dx) >= std::fabs(dy) ? 0 : 1;
    const int sign = (axis == 0 ? dx : dy) > 0.0 ? 1 : -1;
    const int key = axis * 2 + (sign > 0 ? 1 : 0);
    const int cap = (1 << c->run_bits) - 1;
    if (key != c->run_key) {
        cuda_check(xsd::launch_run_field(c->vox.p, c->grid, axis, sign, c->grid.run_shift, cap, c->sm_count,
                                         c->stream),
                   "run field");
        c->run_key = key;
    }
    c->grid.run_axis = axis;
    c->grid.run_sign = sign;
    c->grid.run_mask = cap;
}

void accumulate(xs_context* c, const xs_geometry& g, int angle, const xs_spectrum& spec,
                const xs_sim_config& cfg, uint64_t h0, uint64_t h1, unsigned long long* d_accum,
                xsd::TransportParams* params_only = nullptr)
{
    const xsi::Range range("xscat: scatter transport");
    const auto tA = std::chrono::steady_clock::now();
    require_scene(c);
    const Plan plan = make_plan(g, spec, cfg);
    if (h1 > plan.n_hist)
        h1 = plan.n_hist;
    if (h0 >= h1) {
        c->last = xs_launch_stats{};
        return;
    }
    const int nb = spec.n_bins;
    c->bin_start.reserve(nb + 1);
    c->bin_count.reserve(nb);
    c->bin_e.reserve(nb);
    c->bin_w.reserve(nb);
    c->pool.reserve(1);
    c->status.reserve(1);
    cudaStream_t s = c->stream;
    cuda_check(cudaMemcpyAsync(c->bin_start.p, plan.start.data(), (nb + 1) * 8, cudaMemcpyHostToDevice, s), "H2D");
    cuda_check(cudaMemcpyAsync(c->bin_count.p, plan.counts.data(), nb * 8, cudaMemcpyHostToDevice, s), "H2D");
    cuda_check(cudaMemcpyAsync(c->bin_e.p, spec.energy_kev, nb * 8, cudaMemcpyHostToDevice, s), "H2D");
    cuda_check(cudaMemcpyAsync(c->bin_w.p, spec.weight, nb * 8, cudaMemcpyHostToDevice, s), "H2D");
    cuda_check(cudaMemsetAsync(c->pool.p, 0, 8, s), "memset");
    cuda_check(cudaMemsetAsync(c->status.p, 0, sizeof(xsd::DevStatus), s), "memset");

    ensure_runs(c, xsh::frame_of(g, angle));
    xsd::TransportParams P;
    std::memset(&P, 0, sizeof P);
    P.G = c->grid;
    P.tabs = c->tabs.p;
    P.n_mats = c->n_mats;
    P.n_pal = c->n_pal;
    std::memcpy(P.mats, c->mat_desc, sizeof P.mats);
    std::memcpy(P.pal_mat, c->pal_mat, sizeof P.pal_mat);
    std::memcpy(P.pal_dens, c->pal_dens, sizeof P.pal_dens);
    P.resp_deposit = c->resp_desc;
    const xsh::Frame f = xsh::frame_of(g, angle);
    for (int a = 0; a < 3; ++a) {
        P.src[a] = f.src[a];
        P.center[a] = f.center[a];
        P.uaxis[a] = f.uaxis[a];
        P.normal[a] = f.normal[a];
    }
    P.nu = g.nu;
    P.nv = g.nv;
    P.pitch = g.pixel_pitch;
    P.det_area = g.nu * g.nv * g.pixel_pitch * g.pixel_pitch; // REF detector_area()
    P.n_pixels = static_cast<double>(g.nu) * g.nv;
    P.n_bins = nb;
    P.bin_energy = c->bin_e.p;
    P.bin_weight = c->bin_w.p;
    P.bin_start = c->bin_start.p;
    P.bin_count = c->bin_count.p;
    P.k0 = static_cast<uint32_t>(cfg.seed);
    P.k1 = static_cast<uint32_t>(cfg.seed >> 32);
    P.angle = static_cast<uint32_t>(angle);
    P.splitting = cfg.splitting;
    P.survival = cfg.roulette_survival;
    P.wmin_rel = cfg.roulette_wmin_rel;
    P.step_voxels = cfg.step_voxels;
    P.max_inter = cfg.max_interactions;
    P.track_var = cfg.track_variance ? 1 : 0;
    P.skip = c->macro_skip == 2 ? (c->skip_pays ? 1 : 0) : c->macro_skip;
    if (P.step_voxels > 1) // march mode: the free paths' block walk without runs
        P.G.run_mask = 0;
    { // shared energy knots of the mu tables (REF bundle: yes)
        int first = -1;
        bool same = true;
        for (int m = 1; m < c->n_mats; ++m) {
            if (c->mats[m].t[0].x.empty())
                continue;
            if (first < 0)
                first = m;
            else if (c->mats[m].t[0].x != c->mats[first].t[0].x)
                same = false;
        }
        P.shared_mu_grid = first > 0 && same;
        P.grid_mat = first > 0 ? first : 0;
        // ... and of every energy table (mu, sigma_incoh, sigma_coh, sigma_pe)
        bool all = P.shared_mu_grid != 0;
        for (int m = 1; m < c->n_mats && all; ++m)
            if (!c->mats[m].t[0].x.empty())
                for (int k = 1; k < 4; ++k)
                    all = all && c->mats[m].t[k].x == c->mats[first].t[0].x;
        P.shared_e_grid = all;
    }
    P.march_h = cfg.step_voxels *
                std::min({c->grid.hx, c->grid.hy, c->grid.hz}); // REF trace.cpp:117
    P.march_ih = 1.0 / P.march_h;
    P.accum = d_accum;
    P.off_image = plan.layout.off_image;
    P.off_var = plan.layout.off_variance;
    P.off_bins = plan.layout.off_bins;
    P.off_ledger = plan.layout.off_ledger;
    P.off_diag = plan.layout.off_diag;
    P.log2_img = plan.units.log2_img;
    P.log2_w = plan.units.log2_w;
    P.h_begin = h0;
    P.h_end = h1;
    P.pool = c->pool.p;
    P.grab = c->grab;
    P.status = c->status.p;
    if (params_only) { // a scan group runs this projection with others (scan_group)
        *params_only = P;
        return;
    }

    if (c->engine == 1) { // wavefront engine (wavefront.cu)
        uint32_t n_slots = c->wave_slots;
        if (cfg.track_variance) {
            const uint64_t cap = (uint64_t)cfg.splitting * (uint64_t)cfg.max_interactions;
            if (cap > (1u << 20))
                fail(XS_E_UNSUPPORTED, "xscat-gpu: splitting*max_interactions too large for variance tracking");
            P.var_cap = (int32_t)cap;
            // scratch per live history: keep it near 1 GB
            n_slots = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(n_slots, (1ull << 30) / (12 * cap)));
            // wave_run gives each of its pipelines ceil(n / pipes) slots, side by side
            const uint64_t n_use = std::min<uint64_t>(n_slots, h1 - h0) + (uint64_t)c->wave_pipes;
            c->var_pix.reserve(n_use * cap);
            c->var_val.reserve(n_use * cap);
            P.var_pix = c->var_pix.p;
            P.var_val = c->var_val.p;
        }
        if (!c->wave)
            c->wave = xsd::wave_create();
        xsd::WaveInfo info{};
        const auto tB = std::chrono::steady_clock::now();
        cuda_check(xsd::wave_run(c->wave, P, c->sm_count, n_slots, s, &info, c->ev0, c->wave_pipes),
                   "wavefront transport");
        const auto tC = std::chrono::steady_clock::now();
        cuda_check(cudaEventRecord(c->ev1, s), "event");
        check_status(c, angle, &spec);
        if (std::getenv("XSCAT_TIMING")) {
            auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
            std::fprintf(stderr, "[xscat] accumulate: before %.1f ms, wave_run %.1f ms, status %.1f ms\n",
                         ms(tA, tB), ms(tB, tC), ms(tC, std::chrono::steady_clock::now()));
        }
        float ms = 0.f;
        cuda_check(cudaEventElapsedTime(&ms, c->ev0, c->ev1), "event time");
        c->last.kernel_ms = ms;
        c->last.voxel_format = c->grid.fmt;
        c->last.blocks_per_sm = (uint32_t)info.walk_blocks_per_sm;
        c->last.smem_per_block = 0;
        c->last.slots_per_warp = 0;
        c->last.engine = 1;
        c->last.waves = info.waves;
        c->last.live_histories = info.n_slots;
        c->last.walk_ms = info.walk_ms;
        c->last.setup_ms = info.setup_ms;
        c->last.score_ms = info.score_ms;
        c->last.event_ms = info.event_ms;
        c->last.admit_ms = info.admit_ms;
        c->last.launches = info.launches;
        c->last.palette_size = c->n_pal;
        c->last.upload_bytes = c->last_upload_bytes;
        c->last.block_walk = P.skip && c->grid.ubit ? 1u : 0u;
        return;
    }

    // warp-queue geometry (transport.cu): H live histories per warp, sized
    // to the shared-memory budget
    if ((uint64_t)g.nu * (uint64_t)g.nv >= (1ull << 26))
        fail(XS_E_UNSUPPORTED, "xscat-gpu: scatter detector with %lld pixels exceeds 2^26",
             (long long)g.nu * g.nv);
    const int H = xsd::transport_pick_slots(P, c->max_slots, (size_t)c->smem_kb * 1024);
    const int block = xsd::transport_block_size();
    const size_t smem = xsd::transport_smem_bytes(P);
    int per_sm = 0;
    cuda_check(xsd::transport_prepare(P, smem, &per_sm), "transport occupancy");
    if (per_sm < 1)
        fail(XS_E_UNSUPPORTED, "xscat-gpu: transport kernel does not fit (%zu B shared memory)", smem);
    int grid = c->sm_count * per_sm;
    const uint64_t n = h1 - h0; // no more warps than needed for small launches
    const uint64_t warps_needed = (n + H - 1) / H;
    const uint64_t blocks_needed = std::max<uint64_t>(1, (warps_needed + block / 32 - 1) / (block / 32));
    if ((uint64_t)grid > blocks_needed)
        grid = (int)blocks_needed;
    if (cfg.track_variance) {
        const uint64_t cap = (uint64_t)cfg.splitting * (uint64_t)cfg.max_interactions;
        if (cap > (1u << 20))
            fail(XS_E_UNSUPPORTED, "xscat-gpu: splitting*max_interactions too large for variance tracking");
        P.var_cap = (int32_t)cap;
        const size_t entries = (size_t)grid * (block / 32) * H * cap;
        c->var_pix.reserve(entries);
        c->var_val.reserve(entries);
        P.var_pix = c->var_pix.p;
        P.var_val = c->var_val.p;
    }
    cuda_check(cudaEventRecord(c->ev0, s), "event");
    cuda_check(xsd::launch_transport(P, grid, smem, s), "transport launch");
    cuda_check(cudaEventRecord(c->ev1, s), "event");
    check_status(c, angle, &spec);
    float ms = 0.f;
    cuda_check(cudaEventElapsedTime(&ms, c->ev0, c->ev1), "event time");
    c->last.kernel_ms = ms;
    c->last.voxel_format = c->grid.fmt;
    c->last.blocks_per_sm = (uint32_t)per_sm;
    c->last.smem_per_block = (uint32_t)smem;
    c->last.slots_per_warp = (uint32_t)H;
    c->last.engine = 0;
    c->last.waves = 0;
    c->last.live_histories = (uint32_t)((uint64_t)grid * (block / 32) * H);
    c->last.walk_ms = ms;
    c->last.launches = 1;
    c->last.palette_size = c->n_pal;
    c->last.upload_bytes = c->last_upload_bytes;
    c->last.block_walk = P.skip && c->grid.ubit ? 1u : 0u;
}

// SimResult from n_src accumulators (their sum: one per GPU / context of a
// photon-batch split; device pointers readable from c's device, i.e. local
// or peer memory).  The statistics words are summed on the host, the image
// words by the finalize kernel as it dequantizes (reduce and finalize fused).
void finalize(xs_context* c, const xs_geometry& g, const xs_spectrum& spec, const xs_sim_config& cfg,
              const unsigned long long* const* srcs, int n_src, uint64_t h0, uint64_t h1,
              xs_scatter_result* out, double* d_image)
{
    const xsi::Range range("xscat: finalize");
    const Plan plan = make_plan(g, spec, cfg);
    if (h1 > plan.n_hist)
        h1 = plan.n_hist;
    const xs_accum_layout& L = plan.layout;
    cudaStream_t s = c->stream;
    // statistics words (bins, ledger, diag) -> host, summed over the sources
    const size_t tail = L.words - L.off_bins;
    std::vector<uint64_t> stats(tail, 0), part(tail);
    for (int k = 0; k < n_src; ++k) {
        cuda_check(cudaMemcpyAsync(part.data(), srcs[k] + L.off_bins, tail * 8, cudaMemcpyDefault, s), "D2H stats");
        cuda_check(cudaStreamSynchronize(s), "D2H stats");
        for (size_t i = 0; i < tail; ++i)
            stats[i] += part[i];
    }
    xsh::finalize_stats(spec, plan.counts, h0, h1, stats.data(), stats.data() + (L.off_ledger - L.off_bins),
                        plan.units, out);
    const uint64_t* diag = stats.data() + (L.off_diag - L.off_bins);
    c->last.free_path_steps = diag[0];
    c->last.scoring_steps = diag[1];
    c->last.histories = diag[2];
    c->last.scoring_rays = diag[3];
    c->last.interactions = diag[4];
    c->last.walk_iterations = diag[5];
    c->last.walk_lane_slots = diag[6];
    c->last.uniform_iterations = diag[7];

    double* img = d_image;
    if (!img) {
        c->img.reserve(L.n_pixels);
        img = c->img.p;
    }
    double* var = nullptr;
    if (cfg.track_variance) {
        c->var.reserve(L.n_pixels);
        var = c->var.p;
    }
    cuda_check(xsd::launch_finalize_image(srcs, n_src, L.off_image, L.off_variance, L.n_pixels,
                                          plan.units.log2_img, static_cast<double>(out->histories),
                                          cfg.track_variance, img, var, s),
               "finalize launch");
    if (out->image)
        cuda_check(cudaMemcpyAsync(out->image, img, L.n_pixels * 8, cudaMemcpyDeviceToHost, s), "D2H image");
    if (var && out->variance)
        cuda_check(cudaMemcpyAsync(out->variance, var, L.n_pixels * 8, cudaMemcpyDeviceToHost, s),
                   "D2H variance");
    cuda_check(cudaStreamSynchronize(s), "finalize");
}

void finalize(xs_context* c, const xs_geometry& g, const xs_spectrum& spec, const xs_sim_config& cfg,
              const unsigned long long* d_accum, uint64_t h0, uint64_t h1, xs_scatter_result* out,
              double* d_image)
{
    finalize(c, g, spec, cfg, &d_accum, 1, h0, h1, out, d_image);
}

void primary(xs_context* c, const xs_geometry& g, int angle, const xs_spectrum& spec, double* d_image)
{
    const xsi::Range range("xscat: primary");
    require_scene(c);
    const int nb = spec.n_bins, nm = c->n_mats;
    // REF simulate_primary :343-353 (host glibc loglog, exactly REF's values)
    std::vector<double> atten((size_t)nb * nm, 0.0), w(nb), resp(nb);
    for (int b = 0; b < nb; ++b) {
        resp[b] = xsh::linear(c->resp_dep.view(), spec.energy_kev[b]) / spec.energy_kev[b];
        w[b] = spec.weight[b];
        for (int m = 1; m < nm; ++m)
            if (!c->mats[m].t[0].x.empty())
                atten[(size_t)b * nm + m] = xsh::loglog(c->mats[m].t[0].view(), spec.energy_kev[b]);
    }
    c->prim_atten.reserve(atten.size());
    c->prim_w.reserve(nb);
    c->prim_resp.reserve(nb);
    cudaStream_t s = c->stream;
    cuda_check(cudaMemcpyAsync(c->prim_atten.p, atten.data(), atten.size() * 8, cudaMemcpyHostToDevice, s), "H2D");
    cuda_check(cudaMemcpyAsync(c->prim_w.p, w.data(), nb * 8, cudaMemcpyHostToDevice, s), "H2D");
    cuda_check(cudaMemcpyAsync(c->prim_resp.p, resp.data(), nb * 8, cudaMemcpyHostToDevice, s), "H2D");
    xsd::PrimaryParams P;
    std::memset(&P, 0, sizeof P);
    P.G = c->grid;
    P.n_mats = nm;
    P.n_pal = c->n_pal;
    std::memcpy(P.pal_mat, c->pal_mat, sizeof P.pal_mat);
    std::memcpy(P.pal_dens, c->pal_dens, sizeof P.pal_dens);
    const xsh::Frame f = xsh::frame_of(g, angle);
    for (int a = 0; a < 3; ++a) {
        P.src[a] = f.src[a];
        P.center[a] = f.center[a];
        P.uaxis[a] = f.uaxis[a];
    }
    P.nu = g.nu;
    P.nv = g.nv;
    P.pitch = g.pixel_pitch;
    P.n_bins = nb;
    P.atten = c->prim_atten.p;
    P.wresp = c->prim_w.p;
    P.response = c->prim_resp.p;
    P.image = d_image;
    cuda_check(xsd::launch_primary(P, s), "primary launch");
    cuda_check(cudaStreamSynchronize(s), "primary");
}

} // namespace

// ========================================================== extern "C"
extern "C" {

const char* xs_last_error(const xs_context* ctx)
{
    return ctx ? ctx->err.c_str() : xsh::thread_error();
}

int xs_device_count(int32_t* n)
{
    return guard(nullptr, [&] {
        int c = 0;
        cuda_check(cudaGetDeviceCount(&c), "cudaGetDeviceCount");
        *n = c;
    });
}

int xs_ctx_create(int32_t device, xs_context** out)
{
    *out = nullptr;
    return guard(nullptr, [&] {
        int n = 0;
        cuda_check(cudaGetDeviceCount(&n), "cudaGetDeviceCount");
        if (device < 0 || device >= n)
            fail(XS_E_OUT_OF_RANGE, "xs_ctx_create: device %d out of range (%d devices)", device, n);
        cuda_check(cudaSetDevice(device), "cudaSetDevice");
        if (const char* e = std::getenv("XSCAT_STACK"))
            cuda_check(cudaDeviceSetLimit(cudaLimitStackSize, (size_t)std::atoi(e)), "stack limit");
        auto* c = new xs_context();
        c->device = device;
        cudaDeviceProp prop;
        cuda_check(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
        c->sm_count = prop.multiProcessorCount;
        cuda_check(cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking), "stream");
        c->stream = c->own;
        cuda_check(cudaEventCreate(&c->ev0), "event");
        cuda_check(cudaEventCreate(&c->ev1), "event");
        if (const char* e = std::getenv("XSCAT_GRAB"))
            c->grab = std::max(1, std::atoi(e));
        if (const char* e = std::getenv("XSCAT_SMEM_KB"))
            c->smem_kb = std::max(8, std::min(227, std::atoi(e)));
        if (const char* e = std::getenv("XSCAT_SKIP"))
            c->macro_skip = std::max(0, std::min(2, std::atoi(e)));
        if (const char* e = std::getenv("XSCAT_SLOTS"))
            c->max_slots = std::max(1, std::min(64, std::atoi(e)));
        if (const char* e = std::getenv("XSCAT_LEVELS")) { // e.g. "4,16,64"
            std::vector<int> v;
            for (const char* q = e; *q;) {
                const int x = std::atoi(q);
                if (x >= 2 && x <= 256 && (x & (x - 1)) == 0)
                    v.push_back(x);
                while (*q && *q != ',')
                    ++q;
                if (*q == ',')
                    ++q;
            }
            if (!v.empty() && v.size() <= 3)
                c->lvl_edges2 = v;
            else if (v.size() <= 7)
                c->lvl_edges3 = v;
        }
        if (const char* e = std::getenv("XSCAT_P4"))
            c->compact_palette = std::atoi(e) != 0;
        if (const char* e = std::getenv("XSCAT_RUNS"))
            c->runs = std::atoi(e) != 0;
        if (const char* e = std::getenv("XSCAT_ENGINE"))
            c->engine = std::atoi(e) != 0;
        if (const char* e = std::getenv("XSCAT_WAVE_PIPES"))
            c->wave_pipes = std::max(1, std::min(4, std::atoi(e)));
        if (const char* e = std::getenv("XSCAT_WAVE_SLOTS"))
            c->wave_slots = (uint32_t)std::max(1, std::atoi(e));
        *out = c;
    });
}

void xs_ctx_destroy(xs_context* c)
{
    if (!c)
        return;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    for (auto* b : {&c->img, &c->var, &c->pp_a, &c->pp_b, &c->pp_c, &c->pp_k, &c->bin_e, &c->bin_w,
                    &c->prim_atten, &c->prim_w, &c->prim_resp, &c->tabs, &c->var_val})
        b->release();
    c->vox.release();
    c->dens.release();
    c->pin_vox.release();
    c->pin_dens.release();
    c->pin_raw.release();
    c->accum.release();
    c->bin_start.release();
    c->bin_count.release();
    c->pool.release();
    c->status.release();
    c->var_pix.release();
    c->interp_tab.release();
    c->lvl_scratch.release();
    for (int b = 0; b < 2; ++b) {
        c->scan_img[b].release();
        c->scan_pin[b].release();
        if (c->scan_ev[b])
            cudaEventDestroy(c->scan_ev[b]);
        if (c->scan_done[b])
            cudaEventDestroy(c->scan_done[b]);
    }
    for (cudaEvent_t e : c->up_done)
        if (e)
            cudaEventDestroy(e);
    if (c->copy_stream)
        cudaStreamDestroy(c->copy_stream);
    for (auto& b : c->cc_in)
        b.release();
    for (auto* b : {&c->cc_out, &c->cc_tmp, &c->cc_sg, &c->cc_full})
        b->release();
    c->cc_stats.release();
    for (auto* b : {&c->fbp_in, &c->fbp_q, &c->fbp_k, &c->fbp_views})
        b->release();
    c->fbp_vol.release();
    c->seg_ctl.release();
    c->seg_scratch.release();
    c->seg_thr.release();
    c->seg_ids.release();
    c->seg_labels.release();
    c->seg_dens.release();
    c->seg_vol.release();
    c->seg_pal.release();
    c->probe.release();
    for (auto* b : {&c->loop_a, &c->loop_c, &c->loop_scat, &c->loop_prim, &c->loop_flat, &c->loop_ncc})
        b->release();
    c->loop_vol[0].release();
    c->loop_vol[1].release();
    xsi::mgpu_release(c);
    xsd::wave_destroy(c->wave);
    if (c->ev0)
        cudaEventDestroy(c->ev0);
    if (c->ev1)
        cudaEventDestroy(c->ev1);
    if (c->own)
        cudaStreamDestroy(c->own);
    delete c;
}

int xs_ctx_set_stream(xs_context* c, void* stream)
{
    return guard(c, [&] { c->stream = stream ? static_cast<cudaStream_t>(stream) : c->own; });
}

int xs_ctx_set_option(xs_context* c, const char* key, int64_t value)
{
    return guard(c, [&] {
        const std::string k = key ? key : "";
        if (k == "exact_walk") {
            c->macro_skip = value ? 0 : 1;
        } else if (k == "upload_path") { // 0 host encode, 1 staged H2D + device encode (default)
            c->upload_path = value ? 1 : 0;
        } else if (k == "walk_mode") { // 0 voxel walk, 1 block walk, 2 per phantom (default)
            c->macro_skip = (int)std::max<int64_t>(0, std::min<int64_t>(2, value));
        } else if (k == "smem_kb") {
            c->smem_kb = (int)std::max<int64_t>(8, std::min<int64_t>(227, value));
        } else if (k == "max_slots") {
            c->max_slots = (int)std::max<int64_t>(1, std::min<int64_t>(64, value));
        } else if (k == "grab") {
            c->grab = (int)std::max<int64_t>(1, value);
        } else if (k == "engine") {
            c->engine = value != 0;
        } else if (k == "compact_palette") {
            c->compact_palette = value != 0;
        } else if (k == "runs") { // run field of the block walk (P8); applies at the next upload
            c->runs = value != 0;
        } else if (k == "wave_pipes") {
            c->wave_pipes = (int)std::max<int64_t>(1, std::min<int64_t>(4, value));
        } else if (k == "scan_jobs") { // angles per engine run in device scans (1: one at a time)
            c->scan_jobs = (int)std::max<int64_t>(1, std::min<int64_t>(xs_context::kMaxScanJobs, value));
        } else if (k == "wave_slots") {
            c->wave_slots = (uint32_t)std::max<int64_t>(1, std::min<int64_t>(1 << 25, value));
        } else {
            fail(XS_E_INVALID_ARGUMENT, "xs_ctx_set_option: unknown option '%s'", k.c_str());
        }
    });
}

int xs_ctx_synchronize(xs_context* c)
{
    return guard(c, [&] { cuda_check(cudaStreamSynchronize(c->stream), "synchronize"); });
}

// REF validate_phantom + the device encoding of the grid.  on_device: the
// phantom's id / density arrays are device pointers (the segmentation stage
// builds them in HBM): validation, palette discovery and encoding run on the
// device (segment.cu) and give the same grid as the host path.
static void upload_phantom_impl(xs_context* c, const xs_phantom* ph, bool on_device)
{
    {
        if (ph->dims[0] <= 0 || ph->dims[1] <= 0 || ph->dims[2] <= 0)
            fail(XS_E_RUNTIME, "phantom: dims must be positive");
        if (!(ph->voxel_size[0] > 0.0 && ph->voxel_size[1] > 0.0 && ph->voxel_size[2] > 0.0))
            fail(XS_E_RUNTIME, "phantom: voxel size must be positive");
        if (ph->n_materials <= 0 || !ph->materials)
            fail(XS_E_RUNTIME, "phantom: no material table");
        if (ph->n_materials > xsd::kMaxMaterials)
            fail(XS_E_UNSUPPORTED, "xscat-gpu: at most %d materials (incl. vacuum) supported",
                 xsd::kMaxMaterials);
        const size_t nvox = (size_t)ph->dims[0] * ph->dims[1] * ph->dims[2];
        if (nvox > (size_t)1 << 32)
            fail(XS_E_UNSUPPORTED, "xscat-gpu: at most 2^32 voxels supported");
        std::vector<int> has_tables(ph->n_materials, 0);
        for (int m = 1; m < ph->n_materials; ++m)
            has_tables[m] = ph->materials[m].mu.n > 0;
        ScanResult scan;
        const bool timing = std::getenv("XSCAT_TIMING") != nullptr;
        auto now = [] { return std::chrono::steady_clock::now(); };
        auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
        const auto t0 = now();
        if (on_device) {
            uint32_t tab_bits = 0;
            for (int m = 1; m < ph->n_materials; ++m)
                tab_bits |= has_tables[m] ? (1u << m) : 0u;
            c->seg_ctl.reserve(xsd::seg_ctl_bytes());
            cuda_check(xsd::launch_seg_reset(c->seg_ctl.p, c->stream), "phantom scan");
            cuda_check(xsd::launch_phantom_scan(ph->material_id, ph->density, nvox, ph->n_materials, tab_bits,
                                                c->seg_ctl.p, c->sm_count, c->stream),
                       "phantom scan");
            std::vector<unsigned char> ctl(xsd::seg_ctl_bytes());
            cuda_check(cudaMemcpyAsync(ctl.data(), c->seg_ctl.p, ctl.size(), cudaMemcpyDeviceToHost, c->stream),
                       "phantom scan");
            cuda_check(cudaStreamSynchronize(c->stream), "phantom scan");
            SegCtlView v(ctl.data());
            if (v.first_bad() != ~0ull) {
                uint8_t id = 0;
                float d = 0.f;
                cuda_check(cudaMemcpy(&id, ph->material_id + v.first_bad(), 1, cudaMemcpyDeviceToHost), "D2H");
                cuda_check(cudaMemcpy(&d, ph->density + v.first_bad(), 4, cudaMemcpyDeviceToHost), "D2H");
                fail(XS_E_RUNTIME, "%s", voxel_error(*ph, has_tables, id, d).c_str());
            }
            v.pairs(scan.pairs);
        } else {
            scan_phantom(*ph, has_tables, scan);
        }
        const auto t1 = now();
        if (scan.first_bad != SIZE_MAX)
            fail(XS_E_RUNTIME, "%s", scan.bad_msg.c_str());

        const int n_pairs = (int)scan.pairs.size();
        // 8-bit palette by default: room for three uniform-block level bits
        // (C3: -11% walker iterations, +6% throughput against the 4-bit one)
        const int fmt = (n_pairs <= 8 && c->compact_palette) ? xsd::kFmtP4
                                                              : (n_pairs <= 255 ? xsd::kFmtP8 : xsd::kFmtRaw);
        xsd::Grid G{};
        G.nx = ph->dims[0];
        G.ny = ph->dims[1];
        G.nz = ph->dims[2];
        G.nbx = (G.nx + 3) / 4;
        G.nby = (G.ny + 3) / 4;
        G.nbz = (G.nz + 3) / 4;
        G.ox = ph->origin[0];
        G.oy = ph->origin[1];
        G.oz = ph->origin[2];
        G.hx = ph->voxel_size[0];
        G.hy = ph->voxel_size[1];
        G.hz = ph->voxel_size[2];
        G.ihx = 1.0 / G.hx;
        G.ihy = 1.0 / G.hy;
        G.ihz = 1.0 / G.hz;
        // REF VoxelPhantom::extent: dims * voxel_size, then origin + extent
        G.ux = G.ox + G.nx * G.hx;
        G.uy = G.oy + G.ny * G.hy;
        G.uz = G.oz + G.nz * G.hz;
        G.fmt = fmt;
        G.n_codes = fmt == xsd::kFmtRaw ? 0 : n_pairs;

        const size_t n_bricks = (size_t)G.nbx * G.nby * G.nbz;
        const size_t vox_bytes = n_bricks * (fmt == xsd::kFmtP4 ? 32 : 64);
        const size_t dens_count = fmt == xsd::kFmtRaw ? n_bricks * 64 : 0;
        if (!on_device) {
            c->pin_vox.reserve(vox_bytes);
            c->pin_dens.reserve(std::max<size_t>(dens_count, 1));
            encode_phantom(*ph, fmt, scan.pairs, c->pin_vox.p, c->pin_dens.p, G.nbx, G.nby, G.nbz);
        }
        const auto t2 = now();

        // Uniform blocks: every voxel of an aligned uniform block (all voxels
        // the same code, wholly inside the grid) carries the level of the
        // largest such block holding it, so the walker crosses the block in
        // one step.  Block edges: 4 (a brick) and up, powers of two.
        G.ubit = 0;
        G.lvl_shift = 0;
        G.lvl_log2 = 0;
        std::vector<int> lvl_edges;
        {
            int need = 0; // bits of the palette index
            while ((1 << need) < n_pairs)
                ++need;
            const int width = fmt == xsd::kFmtP4 ? 4 : (fmt == xsd::kFmtP8 ? 8 : 0);
            const int lvl_bits = std::max(0, std::min(3, width - need));
            std::vector<int> edges;
            if (lvl_bits == 1)
                edges = {c->lvl_edge1};
            else if (lvl_bits == 2)
                edges = c->lvl_edges2;
            else if (lvl_bits == 3)
                edges = c->lvl_edges3;
            // runs: the spare bits between the palette index and the level
            const int run_bits =
                (fmt == xsd::kFmtP8 && c->runs && lvl_bits == 3) ? std::min(3, width - need - lvl_bits) : 0;
            const int code_bits = width - lvl_bits;
            G.lvl_shift = code_bits;
            G.ubit = lvl_bits ? (((1 << lvl_bits) - 1) << code_bits) : 0;
            G.run_shift = code_bits - run_bits;
            G.ubit |= ((1 << run_bits) - 1) << G.run_shift;
            c->run_bits = run_bits;
            c->run_key = -1;
            for (size_t l = 0; l < edges.size(); ++l) {
                int lg = 0;
                while ((1 << lg) < edges[l])
                    ++lg;
                G.lvl_log2 |= (uint32_t)lg << (4 * (l + 1));
            }
            lvl_edges = edges;
        }

        c->n_pal = fmt == xsd::kFmtRaw ? 0 : n_pairs;
        std::memset(c->pal_mat, 0, sizeof c->pal_mat);
        std::memset(c->pal_dens, 0, sizeof c->pal_dens);
        for (int k = 0; k < c->n_pal; ++k) {
            c->pal_mat[k] = scan.pairs[k].id;
            std::memcpy(&c->pal_dens[k], &scan.pairs[k].dens_bits, 4);
        }
        c->vox.reserve(vox_bytes);
        if (fmt == xsd::kFmtRaw)
            c->dens.reserve(dens_count);
        if (on_device) {
            std::vector<unsigned long long> keys(scan.pairs.size());
            for (size_t k = 0; k < keys.size(); ++k)
                keys[k] = ((unsigned long long)scan.pairs[k].id << 32) | scan.pairs[k].dens_bits;
            const int n_keys = fmt == xsd::kFmtRaw ? 0 : (int)keys.size();
            c->seg_pal.reserve(std::max(n_keys, 1));
            if (n_keys)
                cuda_check(cudaMemcpyAsync(c->seg_pal.p, keys.data(), n_keys * 8, cudaMemcpyHostToDevice, c->stream),
                           "palette");
            cuda_check(xsd::launch_phantom_encode(ph->material_id, ph->density, c->seg_pal.p, n_keys, G, fmt, c->vox.p,
                                                  fmt == xsd::kFmtRaw ? c->dens.p : nullptr, c->sm_count, c->stream),
                       "encode phantom");
        } else {
            cuda_check(cudaMemcpyAsync(c->vox.p, c->pin_vox.p, vox_bytes, cudaMemcpyHostToDevice, c->stream),
                       "upload voxels");
            if (fmt == xsd::kFmtRaw)
                cuda_check(cudaMemcpyAsync(c->dens.p, c->pin_dens.p, dens_count * 4, cudaMemcpyHostToDevice,
                                           c->stream),
                           "upload densities");
        }
        if (!lvl_edges.empty()) { // uniform-block levels, on the device (levels.cu)
            c->lvl_scratch.reserve(xsd::levels_scratch_bytes(G, lvl_edges.data(), (int)lvl_edges.size()));
            cuda_check(xsd::launch_mark_levels(c->vox.p, G, fmt, lvl_edges.data(), (int)lvl_edges.size(),
                                               c->lvl_scratch.p, c->sm_count, c->stream),
                       "uniform-block levels");
        }
        c->last_upload_bytes = on_device ? 0 : vox_bytes + dens_count * 4;
        cuda_check(cudaStreamSynchronize(c->stream), "upload phantom");
        if (timing)
            std::fprintf(stderr, "[xscat] upload: scan %.1f ms, encode %.1f ms, levels+H2D %.1f ms\n", ms(t0, t1),
                         ms(t1, t2), ms(t2, now()));
        G.vox = c->vox.p;
        G.dens = fmt == xsd::kFmtRaw ? c->dens.p : nullptr;
        c->grid = G;
        c->skip_pays = false;
        if (fmt != xsd::kFmtRaw && G.ubit) { // does crossing uniform blocks pay on this grid?
            xsd::TransportParams P{};
            P.G = G;
            for (int k = 0; k < n_pairs && k < xsd::kMaxPalette; ++k)
                P.pal_mat[k] = scan.pairs[k].id;
            c->probe.reserve(2);
            cuda_check(xsd::launch_walk_probe(P, c->probe.p, c->stream), "walk probe");
            unsigned long long it[2];
            cuda_check(cudaMemcpyAsync(it, c->probe.p, sizeof it, cudaMemcpyDeviceToHost, c->stream), "D2H");
            cuda_check(cudaStreamSynchronize(c->stream), "walk probe");
            c->skip_pays = (double)it[1] < 0.5 * (double)it[0]; // a block step costs ~2 (4-bit) voxel steps
        }
        const bool block_walk = c->macro_skip == 1 || (c->macro_skip == 2 && c->skip_pays);
        if (!block_walk && fmt == xsd::kFmtP8 && n_pairs <= 16) {
            // The voxel walk never reads level bits: re-encode as 4-bit codes.
            // Half the bytes keeps the grid L2-resident for the random voxel
            // reads of speckled phantoms (same palette indices: same results).
            G.fmt = xsd::kFmtP4;
            G.ubit = 0;
            G.lvl_shift = 4;
            G.lvl_log2 = 0;
            c->run_bits = 0;
            const size_t vb4 = n_bricks * 32;
            if (on_device) {
                cuda_check(xsd::launch_phantom_encode(ph->material_id, ph->density, c->seg_pal.p, n_pairs, G,
                                                      xsd::kFmtP4, c->vox.p, nullptr, c->sm_count, c->stream),
                           "encode phantom");
            } else {
                encode_phantom(*ph, xsd::kFmtP4, scan.pairs, c->pin_vox.p, c->pin_dens.p, G.nbx, G.nby, G.nbz);
                cuda_check(cudaMemcpyAsync(c->vox.p, c->pin_vox.p, vb4, cudaMemcpyHostToDevice, c->stream),
                           "upload voxels");
                c->last_upload_bytes += vb4;
            }
            cuda_check(cudaStreamSynchronize(c->stream), "upload phantom");
            c->grid = G;
        }
        c->n_mats = ph->n_materials;
        c->mats.assign(ph->n_materials, HMat{});
        for (int m = 0; m < ph->n_materials; ++m) {
            const xs_material& src = ph->materials[m];
            HMat& d = c->mats[m];
            d.name = src.name ? src.name : (m == 0 ? "vacuum" : "?");
            d.z_eff = src.z_eff;
            d.density_ref = src.density_ref;
            if (m == 0 || src.mu.n <= 0)
                continue;
            d.t[0].set(src.mu);
            d.t[1].set(src.sigma_incoh);
            d.t[2].set(src.sigma_coh);
            d.t[3].set(src.sigma_pe);
            d.t[4].set(src.s_factor);
            d.t[5].set(src.f_factor);
        }
        rebuild_tables(c);
        c->have_phantom = true;
    }
}

// Host arrays through pinned staging (arrays the caller page-locked are
// copied directly): a ring of pinned buffers; worker
// threads copy their share of a chunk of the id / density arrays into the
// chunk's buffer, and the last one to finish queues its DMA, while the others
// go on to the next chunk.  Only the first chunk's copy is not hidden behind
// a DMA (C3 512^3: 19.3 ms, against 21.7 with two 160 MB halves and threads
// spawned per chunk).  Then the device validates and encodes (segment.cu):
// ~2x faster than encoding on the host, and the same device grid.
static void upload_phantom_staged(xs_context* c, const xs_phantom* ph)
{
    if (ph->dims[0] <= 0 || ph->dims[1] <= 0 || ph->dims[2] <= 0 || !ph->material_id || !ph->density) {
        upload_phantom_impl(c, ph, false); // (its checks raise REF's errors)
        return;
    }
    constexpr int kRing = 4;
    const size_t n = (size_t)ph->dims[0] * ph->dims[1] * ph->dims[2];
    auto pinned = [](const void* p) {
        cudaPointerAttributes a{};
        if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        return a.type == cudaMemoryTypeHost;
    };
    if (pinned(ph->material_id) && pinned(ph->density)) { // page-locked by the caller: straight DMA
        c->seg_ids.reserve(n);
        c->seg_dens.reserve(n);
        cuda_check(cudaMemcpyAsync(c->seg_ids.p, ph->material_id, n, cudaMemcpyHostToDevice, c->stream), "H2D");
        cuda_check(cudaMemcpyAsync(c->seg_dens.p, ph->density, n * 4, cudaMemcpyHostToDevice, c->stream), "H2D");
        xs_phantom dp = *ph;
        dp.material_id = c->seg_ids.p;
        dp.density = c->seg_dens.p;
        upload_phantom_impl(c, &dp, true);
        c->last_upload_bytes = n * 5;
        return;
    }
    const size_t chunk = std::min(n, (size_t)8 << 20); // voxels per chunk (40 MB of ids + densities)
    c->seg_ids.reserve(n);
    c->seg_dens.reserve(n);
    // per buffer: the ids, padded to 16 bytes so the densities after them stay aligned
    const size_t id_bytes = (chunk + 15) & ~(size_t)15;
    const size_t buf = id_bytes + 4 * chunk;
    c->pin_raw.reserve(kRing * buf);
    if (!c->copy_stream)
        cuda_check(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking), "stream");
    for (cudaEvent_t& e : c->up_done)
        if (!e)
            cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    // the DMAs into seg_ids / seg_dens run on copy_stream: order them after
    // whatever the context's stream still has queued on those buffers
    cuda_check(cudaEventRecord(c->up_done[0], c->stream), "event");
    cuda_check(cudaStreamWaitEvent(c->copy_stream, c->up_done[0], 0), "event");
    const size_t n_chunks = (n + chunk - 1) / chunk;
    const unsigned nt = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    std::atomic<unsigned> arrived[kRing];
    std::atomic<size_t> issued[kRing]; // chunks queued from each buffer so far
    for (int b = 0; b < kRing; ++b) {
        arrived[b] = 0;
        issued[b] = 0;
    }
    std::atomic<int> err{0};
    auto worker = [&](unsigned t) {
        if (cudaSetDevice(c->device) != cudaSuccess) {
            err = 1;
            return;
        }
        for (size_t k = 0; k < n_chunks && !err; ++k) {
            const int b = (int)(k % kRing);
            // the buffer's previous chunk: queued, then its DMA done
            while (issued[b].load(std::memory_order_acquire) < k / kRing && !err)
                std::this_thread::yield();
            if (err || (k >= kRing && cudaEventSynchronize(c->up_done[b]) != cudaSuccess)) {
                err = 1;
                return;
            }
            const size_t v0 = k * chunk, nv = std::min(chunk, n - v0);
            uint8_t* ids = c->pin_raw.p + (size_t)b * buf;
            float* dens = reinterpret_cast<float*>(ids + id_bytes);
            const size_t a = nv * t / nt, e = nv * (t + 1) / nt;
            std::memcpy(ids + a, ph->material_id + v0 + a, e - a);
            std::memcpy(dens + a, ph->density + v0 + a, (e - a) * 4);
            if (arrived[b].fetch_add(1, std::memory_order_acq_rel) + 1 == nt) { // the chunk is staged
                arrived[b].store(0, std::memory_order_relaxed);
                if (cudaMemcpyAsync(c->seg_ids.p + v0, ids, nv, cudaMemcpyHostToDevice, c->copy_stream) ||
                    cudaMemcpyAsync(c->seg_dens.p + v0, dens, nv * 4, cudaMemcpyHostToDevice, c->copy_stream) ||
                    cudaEventRecord(c->up_done[b], c->copy_stream))
                    err = 1;
                issued[b].store(k / kRing + 1, std::memory_order_release);
            }
        }
    };
    std::vector<std::thread> th;
    for (unsigned t = 1; t < nt; ++t)
        th.emplace_back(worker, t);
    worker(0);
    for (auto& x : th)
        x.join();
    cuda_check(cudaStreamSynchronize(c->copy_stream), "H2D");
    if (err)
        fail(XS_E_CUDA, "phantom upload: staged H2D failed");
    xs_phantom dp = *ph;
    dp.material_id = c->seg_ids.p;
    dp.density = c->seg_dens.p;
    upload_phantom_impl(c, &dp, true);
    c->last_upload_bytes = n * 5;
}

int xs_upload_phantom(xs_context* c, const xs_phantom* ph)
{
    return guard(c, [&] {
        const xsi::Range range("xscat: upload phantom");
        if (c->upload_path == 1)
            upload_phantom_staged(c, ph);
        else
            upload_phantom_impl(c, ph, false);
    });
}

int xs_upload_phantom_device(xs_context* c, const xs_phantom* ph)
{
    return guard(c, [&] { upload_phantom_impl(c, ph, true); });
}

int xs_upload_response(xs_context* c, const xs_response* r)
{
    return guard(c, [&] {
        if (r->dqe.n <= 0 || r->deposit.n <= 0)
            fail(XS_E_RUNTIME, "detector response: empty table");
        c->resp_dqe.set(r->dqe);
        c->resp_dep.set(r->deposit);
        c->have_response = true;
        rebuild_tables(c);
    });
}

int xs_ctx_copy_scene(xs_context* dst, const xs_context* src)
{
    return guard(dst, [&] {
        if (!src || !src->have_phantom)
            fail(XS_E_RUNTIME, "xscat-gpu: no phantom uploaded (xs_upload_phantom)");
        if (dst == src)
            return;
        const xsd::Grid& G = src->grid;
        const size_t n_bricks = (size_t)G.nbx * G.nby * G.nbz;
        const size_t vox_bytes = n_bricks * (G.fmt == xsd::kFmtP4 ? 32 : 64);
        const size_t dens_count = G.fmt == xsd::kFmtRaw ? n_bricks * 64 : 0;
        // the source's device work (upload, encode, levels) must be complete
        cuda_check(cudaSetDevice(src->device), "cudaSetDevice");
        cuda_check(cudaStreamSynchronize(src->stream), "copy scene");
        cuda_check(cudaSetDevice(dst->device), "cudaSetDevice");
        dst->vox.reserve(vox_bytes);
        cuda_check(cudaMemcpyPeerAsync(dst->vox.p, dst->device, src->vox.p, src->device, vox_bytes, dst->stream),
                   "copy scene");
        if (dens_count) {
            dst->dens.reserve(dens_count);
            cuda_check(cudaMemcpyPeerAsync(dst->dens.p, dst->device, src->dens.p, src->device, dens_count * 4,
                                           dst->stream),
                       "copy scene");
        }
        dst->grid = G;
        dst->grid.vox = dst->vox.p;
        dst->grid.dens = dens_count ? dst->dens.p : nullptr;
        dst->n_mats = src->n_mats;
        dst->mats = src->mats;
        dst->n_pal = src->n_pal;
        std::memcpy(dst->pal_mat, src->pal_mat, sizeof dst->pal_mat);
        std::memcpy(dst->pal_dens, src->pal_dens, sizeof dst->pal_dens);
        dst->skip_pays = src->skip_pays;
        dst->run_bits = src->run_bits;
        dst->run_key = src->run_key;
        dst->last_upload_bytes = 0;
        dst->have_phantom = true;
        if (src->have_response) {
            dst->resp_dqe = src->resp_dqe;
            dst->resp_dep = src->resp_dep;
            dst->have_response = true;
        }
        rebuild_tables(dst); // (synchronises dst's stream)
    });
}

int xs_scatter_accumulate_device(xs_context* c, const xs_geometry* g, int32_t angle,
                                 const xs_spectrum* spec, const xs_sim_config* cfg,
                                 uint64_t h0, uint64_t h1, uint64_t* d_accum)
{
    return guard(c, [&] {
        validate_call(*g, angle, *spec, *cfg, "simulate_scatter");
        accumulate(c, *g, angle, *spec, *cfg, h0, h1, reinterpret_cast<unsigned long long*>(d_accum));
    });
}

int xs_scatter_finalize_device(xs_context* c, const xs_geometry* g, const xs_spectrum* spec,
                               const xs_sim_config* cfg, const uint64_t* d_accum, uint64_t h0,
                               uint64_t h1, xs_scatter_result* out, double* d_image)
{
    return guard(c, [&] {
        xsh::validate_sim_config(*cfg);
        xsh::validate_spectrum(*spec);
        xsh::validate_geometry(*g);
        finalize(c, *g, *spec, *cfg, reinterpret_cast<const unsigned long long*>(d_accum), h0, h1, out,
                 d_image);
    });
}

int xs_simulate_scatter_stats(xs_context* c, const xs_geometry* g, int32_t angle,
                              const xs_spectrum* spec, const xs_sim_config* cfg,
                              xs_scatter_result* out)
{
    return guard(c, [&] {
        validate_call(*g, angle, *spec, *cfg, "simulate_scatter");
        const Plan plan = make_plan(*g, *spec, *cfg);
        c->accum.reserve(plan.layout.words);
        cuda_check(cudaMemsetAsync(c->accum.p, 0, plan.layout.words * 8, c->stream), "memset accum");
        accumulate(c, *g, angle, *spec, *cfg, 0, plan.n_hist, c->accum.p);
        finalize(c, *g, *spec, *cfg, c->accum.p, 0, plan.n_hist, out, nullptr);
    });
}

int xs_primary_device(xs_context* c, const xs_geometry* g, int32_t angle, const xs_spectrum* spec,
                      const xs_sim_config* cfg, double* d_image)
{
    return guard(c, [&] {
        validate_call(*g, angle, *spec, *cfg, "simulate_primary");
        primary(c, *g, angle, *spec, d_image);
    });
}

int xs_simulate_primary(xs_context* c, const xs_geometry* g, int32_t angle, const xs_spectrum* spec,
                        const xs_sim_config* cfg, double* image_host)
{
    return guard(c, [&] {
        validate_call(*g, angle, *spec, *cfg, "simulate_primary");
        const size_t np = (size_t)g->nu * g->nv;
        c->img.reserve(np);
        primary(c, *g, angle, *spec, c->img.p);
        cuda_check(cudaMemcpyAsync(image_host, c->img.p, np * 8, cudaMemcpyDeviceToHost, c->stream), "D2H");
        cuda_check(cudaStreamSynchronize(c->stream), "D2H");
    });
}

// run_scan with device outputs (images stay in HBM for the loop's tail):
// same validation, order and error text as xs_run_scan.
// Several angles of a device scan in one wavefront run (wave_run_jobs): each
// pipeline transports one angle at a time into that angle's accumulator and
// takes the next angle as soon as its current one has drained.  Histories and
// tallies are the same as angle by angle, so the images are bit-identical.
// Returns false, with nothing written, when an angle fails validation or the
// transport raises a device error: the caller then runs the group angle by
// angle, which reports REF's error for the first failing angle.
static bool scan_group(xs_context* c, const xs_geometry& g, const xs_spectrum& spec, const xs_sim_config& cfg,
                       const int32_t* angles, int m, double* d_scatter)
{
    try {
        for (int k = 0; k < m; ++k)
            validate_call(g, angles[k], spec, cfg, "simulate_scatter");
    } catch (const Error&) {
        return false;
    }
    const Plan plan = make_plan(g, spec, cfg);
    if (plan.n_hist == 0)
        return false;
    const size_t np = (size_t)g.nu * g.nv;
    std::vector<xsd::TransportParams> jobs(m);
    for (int k = 0; k < m; ++k) {
        c->job_accum[k].reserve(plan.layout.words);
        cuda_check(cudaMemsetAsync(c->job_accum[k].p, 0, plan.layout.words * 8, c->stream), "memset");
        accumulate(c, g, angles[k], spec, cfg, 0, plan.n_hist, c->job_accum[k].p, &jobs[k]);
    }
    if (!c->wave)
        c->wave = xsd::wave_create();
    xsd::WaveInfo info{};
    cuda_check(xsd::wave_run_jobs(c->wave, jobs.data(), m, c->sm_count, c->wave_slots, c->stream, &info, c->ev0,
                                  c->wave_pipes),
               "wavefront transport");
    cuda_check(cudaEventRecord(c->ev1, c->stream), "event");
    xsd::DevStatus st;
    cuda_check(cudaMemcpyAsync(&st, c->status.p, sizeof st, cudaMemcpyDeviceToHost, c->stream), "status readback");
    cuda_check(cudaStreamSynchronize(c->stream), "kernel execution");
    if (st.code != 0)
        return false;
    float ms = 0.f;
    cuda_check(cudaEventElapsedTime(&ms, c->ev0, c->ev1), "event time");
    if (!d_scatter)
        c->job_img.reserve(np);
    for (int k = 0; k < m; ++k) {
        xs_scatter_result r{};
        finalize(c, g, spec, cfg, c->job_accum[k].p, 0, plan.n_hist, &r, d_scatter ? d_scatter + (size_t)k * np : c->job_img.p);
    }
    c->last.kernel_ms = ms;
    c->last.engine = 1;
    c->last.waves = info.waves;
    c->last.live_histories = info.n_slots;
    c->last.walk_ms = info.walk_ms;
    c->last.launches = info.launches;
    return true;
}

static void scan_device_impl(xs_context* c, const xs_geometry* g, const xs_spectrum* spec, const xs_sim_config* cfg,
                             const int32_t* subset, int32_t n_subset, int32_t what, double* d_primary,
                             double* d_scatter, double* seconds)
{
    if (n_subset <= 0)
        fail(XS_E_RUNTIME, "run_scan: empty angle subset");
    xsh::validate_sim_config(*cfg);
    xsh::validate_geometry(*g);
    for (int i = 0; i < n_subset; ++i)
        if (subset[i] < 0 || subset[i] >= g->n_angles)
            fail(XS_E_OUT_OF_RANGE, "run_scan: angle index %d out of range", subset[i]);
    const bool want_primary = what != 1, want_scatter = what != 0;
    const size_t np = (size_t)g->nu * g->nv;
    // groups of consecutive angles that share the run field (scan_group)
    const bool grouped = want_scatter && c->engine == 1 && c->scan_jobs > 1 && c->wave_pipes > 1 &&
                         !cfg->track_variance && cfg->step_voxels == 1;
    int group_end = 0;  // angles [group_begin, group_end) were transported by a group ...
    int group_begin = 0;
    int single_end = 0; // ... angles before this one go one at a time (their group failed)
    for (int i = 0; i < n_subset; ++i) {
        const auto t0 = std::chrono::steady_clock::now();
        if (grouped && i >= group_end && i >= single_end) {
            int m = 1;
            if (subset[i] >= 0 && subset[i] < g->n_angles) {
                const int key = run_key_of(xsh::frame_of(*g, subset[i]));
                while (m < c->scan_jobs && i + m < n_subset && subset[i + m] >= 0 && subset[i + m] < g->n_angles &&
                       run_key_of(xsh::frame_of(*g, subset[i + m])) == key)
                    ++m;
            }
            bool ok = false;
            if (m > 1) {
                try { // (any failure: the angles go one at a time and report REF's error)
                    ok = scan_group(c, *g, *spec, *cfg, subset + i, m, d_scatter ? d_scatter + (size_t)i * np : nullptr);
                } catch (const Error&) {
                    ok = false;
                }
            }
            if (ok) {
                group_begin = i;
                group_end = i + m;
            } else {
                single_end = i + m;
            }
        }
        const bool in_group = i >= group_begin && i < group_end;
        try {
            if (want_scatter && !in_group) {
                validate_call(*g, subset[i], *spec, *cfg, "simulate_scatter");
                const Plan plan = make_plan(*g, *spec, *cfg);
                c->accum.reserve(plan.layout.words);
                cuda_check(cudaMemsetAsync(c->accum.p, 0, plan.layout.words * 8, c->stream), "memset");
                accumulate(c, *g, subset[i], *spec, *cfg, 0, plan.n_hist, c->accum.p);
                xs_scatter_result r{};
                c->scan_img[0].reserve(np);
                double* dst = d_scatter ? d_scatter + (size_t)i * np : c->scan_img[0].p;
                finalize(c, *g, *spec, *cfg, c->accum.p, 0, plan.n_hist, &r, dst);
            }
            if (want_primary) {
                validate_call(*g, subset[i], *spec, *cfg, "simulate_primary");
                c->img.reserve(np);
                primary(c, *g, subset[i], *spec, d_primary ? d_primary + (size_t)i * np : c->img.p);
                if (seconds)
                    cuda_check(cudaStreamSynchronize(c->stream), "primary");
            }
        } catch (const Error& e) {
            fail(XS_E_RUNTIME, "run_scan: angle index %d: %s", subset[i], e.msg.c_str());
        }
        if (seconds)
            seconds[i] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    }
    cuda_check(cudaStreamSynchronize(c->stream), "run_scan");
}

int xs_run_scan_device(xs_context* c, const xs_geometry* g, const xs_spectrum* spec, const xs_sim_config* cfg,
                       const int32_t* subset, int32_t n_subset, int32_t what, double* d_primary, double* d_scatter,
                       double* seconds)
{
    return guard(c, [&] { scan_device_impl(c, g, spec, cfg, subset, n_subset, what, d_primary, d_scatter, seconds); });
}

int xs_run_scan(xs_context* c, const xs_geometry* g, const xs_spectrum* spec, const xs_sim_config* cfg,
                const int32_t* subset, int32_t n_subset, int32_t what, double* primary_out,
                double* scatter_out, double* seconds)
{
    return guard(c, [&] {
        if (n_subset <= 0)
            fail(XS_E_RUNTIME, "run_scan: empty angle subset");
        xsh::validate_sim_config(*cfg);
        xsh::validate_geometry(*g);
        for (int i = 0; i < n_subset; ++i)
            if (subset[i] < 0 || subset[i] >= g->n_angles)
                fail(XS_E_OUT_OF_RANGE, "run_scan: angle index %d out of range", subset[i]);
        const bool want_primary = what != 1, want_scatter = what != 0;
        const size_t np = (size_t)g->nu * g->nv;
        // Scatter images leave through a copy stream and pinned staging (double
        // buffered): the D2H and the host copy of angle i overlap the
        // transport of angle i + 1.
        if (!c->copy_stream)
            cuda_check(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking), "stream");
        for (int b = 0; b < 2; ++b) {
            if (!c->scan_ev[b])
                cuda_check(cudaEventCreateWithFlags(&c->scan_ev[b], cudaEventDisableTiming), "event");
            if (!c->scan_done[b])
                cuda_check(cudaEventCreateWithFlags(&c->scan_done[b], cudaEventDisableTiming), "event");
        }
        std::thread copier[2];
        auto drain = [&](int b) {
            if (copier[b].joinable())
                copier[b].join();
        };
        struct Joiner {
            std::function<void()> f;
            ~Joiner() { f(); }
        } join_all{[&] {
            drain(0);
            drain(1);
        }};
        // units of one angle, or of a group of consecutive angles transported in
        // one engine run (scan_group); unit u uses image / staging buffer pair u & 1
        const bool grouped = want_scatter && c->engine == 1 && c->scan_jobs > 1 && c->wave_pipes > 1 &&
                             !cfg->track_variance && cfg->step_voxels == 1;
        int single_end = 0; // angles before this one go one at a time (their group failed)
        for (int i = 0, u = 0; i < n_subset; ++u) {
            const auto t0 = std::chrono::steady_clock::now();
            const int b = u & 1;
            int m = 1;
            if (want_scatter) {
                drain(b); // unit u - 2's copy out of this buffer pair
                bool ok = false;
                if (grouped && i >= single_end) {
                    const int key = run_key_of(xsh::frame_of(*g, subset[i]));
                    while (m < c->scan_jobs && i + m < n_subset && run_key_of(xsh::frame_of(*g, subset[i + m])) == key)
                        ++m;
                    if (m > 1) {
                        try { // (any failure: the angles go one at a time and report REF's error)
                            c->scan_img[b].reserve((size_t)m * np);
                            ok = scan_group(c, *g, *spec, *cfg, subset + i, m, c->scan_img[b].p);
                        } catch (const Error&) {
                            ok = false;
                        }
                        if (!ok) {
                            single_end = i + m;
                            m = 1;
                        }
                    }
                }
                if (!ok) {
                    try {
                        validate_call(*g, subset[i], *spec, *cfg, "simulate_scatter");
                        const Plan plan = make_plan(*g, *spec, *cfg);
                        c->accum.reserve(plan.layout.words);
                        cuda_check(cudaMemsetAsync(c->accum.p, 0, plan.layout.words * 8, c->stream), "memset");
                        accumulate(c, *g, subset[i], *spec, *cfg, 0, plan.n_hist, c->accum.p);
                        xs_scatter_result r{};
                        c->scan_img[b].reserve(np);
                        finalize(c, *g, *spec, *cfg, c->accum.p, 0, plan.n_hist, &r, c->scan_img[b].p);
                    } catch (const Error& e) {
                        fail(XS_E_RUNTIME, "run_scan: angle index %d: %s", subset[i], e.msg.c_str());
                    }
                }
                if (scatter_out) {
                    const size_t n_img = (size_t)m * np;
                    c->scan_pin[b].reserve(n_img);
                    cuda_check(cudaEventRecord(c->scan_ev[b], c->stream), "event");
                    cuda_check(cudaStreamWaitEvent(c->copy_stream, c->scan_ev[b], 0), "wait");
                    cuda_check(cudaMemcpyAsync(c->scan_pin[b].p, c->scan_img[b].p, n_img * 8, cudaMemcpyDeviceToHost,
                                               c->copy_stream),
                               "D2H image");
                    cuda_check(cudaEventRecord(c->scan_done[b], c->copy_stream), "event");
                    double* dst = scatter_out + (size_t)i * np;
                    const double* src = c->scan_pin[b].p;
                    cudaEvent_t done = c->scan_done[b];
                    copier[b] = std::thread([dst, src, n_img, done] {
                        cudaEventSynchronize(done);
                        std::memcpy(dst, src, n_img * 8);
                    });
                }
                // the next unit's transport overwrites only the accumulators, and
                // its finalize writes the other image buffer
            }
            for (int k = i; k < i + m; ++k) {
                try {
                    if (want_primary) {
                        validate_call(*g, subset[k], *spec, *cfg, "simulate_primary");
                        c->img.reserve(np);
                        primary(c, *g, subset[k], *spec, c->img.p);
                        if (primary_out)
                            cuda_check(cudaMemcpyAsync(primary_out + (size_t)k * np, c->img.p, np * 8,
                                                       cudaMemcpyDeviceToHost, c->stream),
                                       "D2H");
                        cuda_check(cudaStreamSynchronize(c->stream), "D2H");
                    }
                } catch (const Error& e) {
                    fail(XS_E_RUNTIME, "run_scan: angle index %d: %s", subset[k], e.msg.c_str());
                }
            }
            if (seconds) { // a group's time is shared by its angles
                const double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
                for (int k = i; k < i + m; ++k)
                    seconds[k] = dt / m;
            }
            i += m;
        }
    });
}

int xs_last_launch_stats(const xs_context* c, xs_launch_stats* out)
{
    *out = c->last;
    return XS_OK;
}

// ------------------------------------------------------------ postprocess
namespace {
// REF sg_smooth set-up (postprocess.cpp:124-145): validation and the
// (half+1)^2 truncated kernels (host-solved by REF's normal equations).
int upload_sg_kernels(xs_context* c, int nu, int nv, int window, int polyorder)
{
    xsh::validate_sg(window, polyorder);
    if (nu < window || nv < window)
        fail(XS_E_RUNTIME, "sg_smooth: image dims smaller than filter window");
    const int half = window / 2, W = 2 * half + 1;
    std::vector<double> K((size_t)(half + 1) * (half + 1) * W, 0.0);
    for (int l = 0; l <= half; ++l)
        for (int r = 0; r <= half; ++r) {
            const auto k = xsh::sg_kernel(l, r, polyorder);
            std::copy(k.begin(), k.end(), K.begin() + (size_t)(l * (half + 1) + r) * W);
        }
    c->pp_k.reserve(K.size());
    cuda_check(cudaMemcpyAsync(c->pp_k.p, K.data(), K.size() * 8, cudaMemcpyHostToDevice, c->stream), "H2D");
    return half;
}

// REF interpolate_angles bracket selection (postprocess.cpp:147-196), on the
// host; the per-pixel lerp runs on the device.
void upload_interp_plan(xs_context* c, const double* src, int n_src, const double* tgt, int n_tgt)
{
    for (int i = 1; i < n_src; ++i)
        if (!(src[i] > src[i - 1]))
            fail(XS_E_RUNTIME, "interpolate_angles: source angles not sorted");
    for (int i = 1; i < n_tgt; ++i)
        if (!(tgt[i] > tgt[i - 1]))
            fail(XS_E_RUNTIME, "interpolate_angles: target angles not sorted");
    std::vector<xsd::InterpEntry> tab(n_tgt);
    const double period = 2.0 * kPi;
    for (int t = 0; t < n_tgt; ++t) {
        const double b = tgt[t];
        const double* lb = std::lower_bound(src, src + n_src, b);
        if (lb != src + n_src && *lb == b) {
            tab[t] = {(int)(lb - src), (int)(lb - src), 1, 0.0};
            continue;
        }
        if (n_src < 2)
            fail(XS_E_RUNTIME, "interpolate_angles: missing bracket for angle %f", b);
        int hi = (int)(lb - src), lo;
        double a_lo, a_hi;
        if (hi == 0) {
            lo = n_src - 1;
            a_lo = src[lo] - period;
            a_hi = src[0];
        } else if (hi == n_src) {
            lo = n_src - 1;
            hi = 0;
            a_lo = src[lo];
            a_hi = src[0] + period;
        } else {
            lo = hi - 1;
            a_lo = src[lo];
            a_hi = src[hi];
        }
        tab[t] = {lo, hi, 0, (b - a_lo) / (a_hi - a_lo)};
    }
    if (n_tgt == 0)
        return;
    c->interp_tab.reserve(n_tgt);
    cuda_check(cudaMemcpyAsync(c->interp_tab.p, tab.data(), n_tgt * sizeof(xsd::InterpEntry),
                               cudaMemcpyHostToDevice, c->stream),
               "H2D");
}

struct Staged {
    const double* in;
    double* out;
};

// Host-pointer mode: stage through context buffers.
Staged stage(xs_context* c, const double* in, size_t n_in, double* out, size_t n_out, bool device)
{
    if (device)
        return {in, out};
    c->pp_a.reserve(n_in);
    c->pp_b.reserve(n_out);
    cuda_check(cudaMemcpyAsync(c->pp_a.p, in, n_in * 8, cudaMemcpyHostToDevice, c->stream), "H2D");
    return {c->pp_a.p, c->pp_b.p};
}

void unstage(xs_context* c, const Staged& s, double* out, size_t n_out, bool device)
{
    if (!device)
        cuda_check(cudaMemcpyAsync(out, s.out, n_out * 8, cudaMemcpyDeviceToHost, c->stream), "D2H");
    cuda_check(cudaStreamSynchronize(c->stream), "postprocess");
}
} // namespace

int xs_sg_smooth(xs_context* c, const double* in, double* out, int32_t nu, int32_t nv, int32_t n_images,
                 int32_t window, int32_t polyorder, int32_t device_ptrs)
{
    return guard(c, [&] {
        const int half = upload_sg_kernels(c, nu, nv, window, polyorder);
        const size_t n = (size_t)nu * nv * n_images;
        const Staged s = stage(c, in, n, out, n, device_ptrs != 0);
        c->pp_c.reserve(n);
        cuda_check(xsd::launch_sg(s.in, c->pp_c.p, s.out, nu, nv, n_images, half, c->pp_k.p, c->stream), "sg");
        unstage(c, s, out, n, device_ptrs != 0);
    });
}

int xs_interpolate_angles(xs_context* c, const double* in, const double* src, int32_t n_src, double* out,
                          const double* tgt, int32_t n_tgt, int32_t nu, int32_t nv, int32_t device_ptrs)
{
    return guard(c, [&] {
        upload_interp_plan(c, src, n_src, tgt, n_tgt);
        if (n_tgt == 0)
            return;
        const size_t np = (size_t)nu * nv;
        const Staged s = stage(c, in, np * n_src, out, np * n_tgt, device_ptrs != 0);
        cuda_check(xsd::launch_interp(s.in, s.out, c->interp_tab.p, n_tgt, np, c->stream), "interp");
        unstage(c, s, out, np * n_tgt, device_ptrs != 0);
    });
}

int xs_upsample_image(xs_context* c, const double* in, int32_t nu, int32_t nv, int32_t n_images,
                      double* out, int32_t nu_out, int32_t nv_out, int32_t device_ptrs)
{
    return guard(c, [&] {
        if (nu_out < nu || nv_out < nv)
            fail(XS_E_RUNTIME, "upsample_image: target dims must be >= source dims");
        if (nu < 1 || nv < 1)
            fail(XS_E_RUNTIME, "upsample_image: degenerate source");
        const size_t n_in = (size_t)nu * nv * n_images, n_out = (size_t)nu_out * nv_out * n_images;
        const Staged s = stage(c, in, n_in, out, n_out, device_ptrs != 0);
        c->pp_c.reserve((size_t)nu_out * nv * n_images);
        cuda_check(xsd::launch_upsample(s.in, c->pp_c.p, s.out, nu, nv, n_images, nu_out, nv_out, c->stream),
                   "upsample");
        unstage(c, s, out, n_out, device_ptrs != 0);
    });
}

int xs_downsample_average(xs_context* c, const double* in, int32_t nu, int32_t nv, int32_t n_images,
                          double* out, int32_t nu_out, int32_t nv_out, int32_t device_ptrs)
{
    return guard(c, [&] {
        if (nu_out > nu || nv_out > nv || nu_out < 1 || nv_out < 1)
            fail(XS_E_RUNTIME, "downsample_average: bad target dims");
        const size_t n_in = (size_t)nu * nv * n_images, n_out = (size_t)nu_out * nv_out * n_images;
        const Staged s = stage(c, in, n_in, out, n_out, device_ptrs != 0);
        cuda_check(xsd::launch_downsample(s.in, s.out, nu, nv, n_images, nu_out, nv_out, c->stream),
                   "downsample");
        unstage(c, s, out, n_out, device_ptrs != 0);
    });
}

// ------------------------------------------------- correction-loop stages
namespace {
// host -> device staging of one input (device_ptrs: used in place)
const double* cc_input(xs_context* c, int k, const double* p, size_t n, bool device)
{
    if (device)
        return p;
    c->cc_in[k].reserve(n);
    cuda_check(cudaMemcpyAsync(c->cc_in[k].p, p, n * 8, cudaMemcpyHostToDevice, c->stream), "H2D");
    return c->cc_in[k].p;
}

unsigned long long* cc_stats(xs_context* c, int n_views)
{
    const size_t words = (xsd::correct_stats_bytes(n_views) + 7) / 8;
    c->cc_stats.reserve(words);
    cuda_check(cudaMemsetAsync(c->cc_stats.p, 0, words * 8, c->stream), "memset");
    return c->cc_stats.p;
}

void cc_read_stats(xs_context* c, uint64_t out[5])
{
    cuda_check(cudaMemcpyAsync(out, c->cc_stats.p, 5 * 8, cudaMemcpyDeviceToHost, c->stream), "D2H");
    cuda_check(cudaStreamSynchronize(c->stream), "correction");
}
} // namespace

int xs_intensity_to_attenuation(xs_context* c, const double* intensity, const double* flatfield, int32_t nu,
                                int32_t nv, int32_t n_images, double* out, int32_t device_ptrs)
{
    return guard(c, [&] {
        const bool dev = device_ptrs != 0;
        const size_t np = (size_t)nu * nv, n = np * n_images;
        const double* in = cc_input(c, 0, intensity, n, dev);
        const double* flat = cc_input(c, 1, flatfield, np, dev);
        double* o = out;
        if (!dev) {
            c->cc_out.reserve(n);
            o = c->cc_out.p;
        }
        unsigned long long* st = cc_stats(c, 1);
        cuda_check(xsd::launch_i2a(in, flat, o, np, n_images, st, c->sm_count, c->stream), "intensity_to_attenuation");
        uint64_t h[5];
        cc_read_stats(c, h);
        if (h[1] > 0) // recon.cpp:343-345
            fail(XS_E_RUNTIME, "intensity_to_attenuation: %llu non-positive pixels (underexposed or invalid data)",
                 (unsigned long long)h[1]);
        if (!dev) {
            cuda_check(cudaMemcpyAsync(out, o, n * 8, cudaMemcpyDeviceToHost, c->stream), "D2H");
            cuda_check(cudaStreamSynchronize(c->stream), "D2H");
        }
    });
}

int xs_correct_projections(xs_context* c, const double* a, const double* primary, const double* scatter,
                           int32_t nu, int32_t nv, int32_t n_images, double* out, uint64_t* clamped,
                           int32_t device_ptrs)
{
    return guard(c, [&] {
        const bool dev = device_ptrs != 0;
        const size_t n = (size_t)nu * nv * n_images;
        const double* da = cc_input(c, 0, a, n, dev);
        const double* dp = cc_input(c, 1, primary, n, dev);
        const double* ds = cc_input(c, 2, scatter, n, dev);
        double* o = out;
        if (!dev) {
            c->cc_out.reserve(n);
            o = c->cc_out.p;
        }
        unsigned long long* st = cc_stats(c, 1);
        cuda_check(xsd::launch_correct(da, dp, ds, o, n, st, c->sm_count, c->stream), "correct_projections");
        uint64_t h[5];
        cc_read_stats(c, h);
        if (h[1] > 0) // correction.cpp:72-73
            fail(XS_E_RUNTIME, "correct_projections: non-positive primary pixel");
        if (clamped)
            *clamped = h[0];
        if (!dev) {
            cuda_check(cudaMemcpyAsync(out, o, n * 8, cudaMemcpyDeviceToHost, c->stream), "D2H");
            cuda_check(cudaStreamSynchronize(c->stream), "D2H");
        }
    });
}

int xs_correction_tail(xs_context* c, const double* scatter_sub, const double* sub_angles, int32_t n_sub,
                       const double* primary_mc, const double* full_angles, int32_t n_full, int32_t nu, int32_t nv,
                       int32_t sg_window, int32_t sg_order, const double* a, int32_t nu_out, int32_t nv_out,
                       double* corrected, double* mean_scatter_fraction, uint64_t* clamped, int32_t device_ptrs)
{
    return guard(c, [&] {
        if (nu_out < nu || nv_out < nv)
            fail(XS_E_RUNTIME, "upsample_image: target dims must be >= source dims");
        const bool dev = device_ptrs != 0;
        const size_t np = (size_t)nu * nv, npo = (size_t)nu_out * nv_out;
        // REF correction.cpp:199-205: SG on every scatter image, then angles
        const int half = upload_sg_kernels(c, nu, nv, sg_window, sg_order);
        upload_interp_plan(c, sub_angles, n_sub, full_angles, n_full);
        if (n_full == 0)
            return;
        const double* ds = cc_input(c, 0, scatter_sub, np * n_sub, dev);
        const double* dp = cc_input(c, 1, primary_mc, np * n_full, dev);
        const double* da = cc_input(c, 2, a, npo * n_full, dev);
        c->cc_sg.reserve(np * n_sub);
        c->pp_c.reserve(np * n_sub);
        cuda_check(xsd::launch_sg(ds, c->pp_c.p, c->cc_sg.p, nu, nv, n_sub, half, c->pp_k.p, c->stream), "sg");
        c->cc_full.reserve(np * n_full);
        cuda_check(xsd::launch_interp(c->cc_sg.p, c->cc_full.p, c->interp_tab.p, n_full, np, c->stream), "interp");
        // correction.cpp:206-246, fused (correct.cu)
        double* o = corrected;
        if (!dev) {
            c->cc_out.reserve(npo * n_full);
            o = c->cc_out.p;
        }
        c->cc_tmp.reserve(2 * (size_t)n_full * nv * nu_out);
        unsigned long long* st = cc_stats(c, n_full);
        cuda_check(xsd::launch_correction_tail(dp, c->cc_full.p, da, c->cc_tmp.p, o, nu, nv, n_full, nu_out,
                                               nv_out, st, c->stream),
                   "correction tail");
        uint64_t h[5];
        cc_read_stats(c, h);
        if (h[1] > 0)
            fail(XS_E_RUNTIME, "correct_projections: non-positive primary pixel");
        if (clamped)
            *clamped = h[0];
        if (mean_scatter_fraction) // fixed-point sum of the fractions / count
            *mean_scatter_fraction =
                h[4] ? (std::ldexp((double)h[2], -32) + std::ldexp((double)h[3], -64)) / (double)h[4] : 0.0;
        if (!dev) {
            cuda_check(cudaMemcpyAsync(corrected, o, npo * n_full * 8, cudaMemcpyDeviceToHost, c->stream), "D2H");
            cuda_check(cudaStreamSynchronize(c->stream), "D2H");
        }
    });
}

// ------------------------------------------------------------------- FDK
void xs_default_voxel_size(const xs_geometry* g, const int32_t dims[3], double out[3])
{
    // REF recon.cpp:13-18
    const double fov = g->nu * g->pixel_pitch * g->sod / g->sdd;
    const double h = fov / std::max({dims[0], dims[1], dims[2]});
    out[0] = out[1] = out[2] = h;
}

int xs_fbp_reconstruct(xs_context* c, const double* stack, const double* angles, int32_t n_views, int32_t nu,
                       int32_t nv, const xs_geometry* g, const int32_t dims[3], const double voxel[3],
                       int32_t hann, float* volume, int32_t device_ptrs)
{
    return guard(c, [&] {
        if (n_views <= 0)
            fail(XS_E_RUNTIME, "fbp: empty projection stack");
        // REF recon.cpp:62-67: coverage >= 180 deg + fan, span = 2 pi - largest circular gap
        const double pi = kPi;
        const double fan = 2.0 * std::atan(0.5 * g->nu * g->pixel_pitch / g->sdd);
        double span = 0.0;
        if (n_views >= 2) {
            double max_gap = 2.0 * pi + angles[0] - angles[n_views - 1];
            for (int i = 1; i < n_views; ++i)
                max_gap = std::max(max_gap, angles[i] - angles[i - 1]);
            span = 2.0 * pi - max_gap;
        }
        if (n_views < 2 || span + 1e-9 < pi + fan)
            fail(XS_E_RUNTIME, "fbp: insufficient angular coverage (need >= 180 deg + fan)");
        if (dims[0] <= 0 || dims[1] <= 0 || dims[2] <= 0 || nu < 2 || nv < 2)
            fail(XS_E_RUNTIME, "fbp: degenerate dimensions");
        const double R = g->sod, D = g->sdd;
        const double du = g->pixel_pitch * R / D, dv = du;
        // REF recon.cpp:23-43 ramp kernel (Hann = (1/4, 1/2, 1/4) smoothing of Ram-Lak)
        auto ramlak = [&](int k) -> double {
            if (k == 0)
                return 1.0 / (8.0 * du * du);
            if (k % 2 == 0)
                return 0.0;
            return -1.0 / (2.0 * pi * pi * k * k * du * du);
        };
        std::vector<double> kern(2 * (size_t)nu - 1);
        for (int k = -(nu - 1); k <= nu - 1; ++k) {
            double v = ramlak(k);
            if (hann)
                v = 0.5 * ramlak(k) + 0.25 * (ramlak(k - 1) + ramlak(k + 1));
            kern[k + nu - 1] = v;
        }
        // REF :76-82 per-view angular weights; cos / sin of the view angles (glibc)
        std::vector<double> views(3 * (size_t)n_views);
        for (int i = 0; i < n_views; ++i) {
            const double prev = (i == 0) ? angles[n_views - 1] - 2.0 * pi : angles[i - 1];
            const double next = (i == n_views - 1) ? angles[0] + 2.0 * pi : angles[i + 1];
            views[3 * i + 0] = std::cos(angles[i]);
            views[3 * i + 1] = std::sin(angles[i]);
            views[3 * i + 2] = 0.5 * (next - prev);
        }
        cudaStream_t st = c->stream;
        const size_t np = (size_t)nu * nv * n_views, nvox = (size_t)dims[0] * dims[1] * dims[2];
        const double* in = stack;
        if (!device_ptrs) {
            c->fbp_in.reserve(np);
            cuda_check(cudaMemcpyAsync(c->fbp_in.p, stack, np * 8, cudaMemcpyHostToDevice, st), "H2D");
            in = c->fbp_in.p;
        }
        c->fbp_q.reserve(np);
        c->fbp_k.reserve(kern.size());
        c->fbp_views.reserve(views.size());
        cuda_check(cudaMemcpyAsync(c->fbp_k.p, kern.data(), kern.size() * 8, cudaMemcpyHostToDevice, st), "H2D");
        cuda_check(cudaMemcpyAsync(c->fbp_views.p, views.data(), views.size() * 8, cudaMemcpyHostToDevice, st),
                   "H2D");
        if (xsd::fbp_filter_smem(nu) > 227 * 1024)
            fail(XS_E_UNSUPPORTED, "fbp: detector rows of %d pixels exceed the shared-memory filter", nu);
        cuda_check(xsd::launch_fbp_filter(in, c->fbp_q.p, c->fbp_k.p, nu, nv, n_views, R, du, dv, st), "fbp filter");
        float* vol = volume;
        if (!device_ptrs) {
            c->fbp_vol.reserve(nvox);
            vol = c->fbp_vol.p;
        }
        const int d3[3] = {dims[0], dims[1], dims[2]};
        cuda_check(xsd::launch_fbp_backproject(c->fbp_q.p, c->fbp_views.p, n_views, nu, nv, d3, voxel, R, du, dv,
                                               vol, st),
                   "fbp backprojection");
        if (!device_ptrs)
            cuda_check(cudaMemcpyAsync(volume, vol, nvox * 4, cudaMemcpyDeviceToHost, st), "D2H");
        cuda_check(cudaStreamSynchronize(st), "fbp");
    });
}

// ---------------------------------------------------------- segmentation
// REF otsu_thresholds / segment_volume / to_density_phantom (recon.cpp:159-322)
// and the loop's fused segmentation stage (correction.cpp:167-172) on the
// device (segment.cu); SURVEY.md §8(f) rank 3.
static const float* seg_volume_in(xs_context* c, const float* volume, size_t nvox, int32_t device_ptrs)
{
    if (device_ptrs)
        return volume;
    c->seg_vol.reserve(nvox);
    cuda_check(cudaMemcpyAsync(c->seg_vol.p, volume, nvox * 4, cudaMemcpyHostToDevice, c->stream), "H2D");
    return c->seg_vol.p;
}

static void seg_otsu(xs_context* c, const float* vol, const int32_t dims[3], int n_classes, int bins,
                     double* thresholds)
{
    if (n_classes < 2 || n_classes > 4)
        fail(XS_E_INVALID_ARGUMENT, "otsu: n_classes must be in [2,4]");
    if (bins < n_classes)
        fail(XS_E_INVALID_ARGUMENT, "otsu: too few histogram bins");
    if (dims[0] <= 0 || dims[1] <= 0 || dims[2] <= 0)
        fail(XS_E_RUNTIME, "otsu: degenerate histogram");
    c->seg_ctl.reserve(xsd::seg_ctl_bytes());
    c->seg_scratch.reserve(xsd::otsu_scratch_bytes(bins, n_classes));
    c->seg_thr.reserve(16);
    cuda_check(xsd::launch_seg_reset(c->seg_ctl.p, c->stream), "otsu");
    const int d[3] = {dims[0], dims[1], dims[2]};
    cuda_check(xsd::launch_otsu(vol, d, n_classes, bins, c->seg_ctl.p, c->seg_scratch.p, c->seg_thr.p, c->sm_count,
                                c->stream),
               "otsu");
    unsigned char ctl[64];
    cuda_check(cudaMemcpyAsync(ctl, c->seg_ctl.p, sizeof ctl, cudaMemcpyDeviceToHost, c->stream), "D2H");
    cuda_check(cudaMemcpyAsync(thresholds, c->seg_thr.p, (n_classes - 1) * sizeof(double), cudaMemcpyDeviceToHost,
                               c->stream),
               "D2H");
    cuda_check(cudaStreamSynchronize(c->stream), "otsu");
    if (SegCtlView(ctl).status() != 0)
        fail(XS_E_RUNTIME, "otsu: degenerate histogram");
}

static void check_thresholds(const double* thr, int n_thr, int n_class_map)
{
    for (int i = 1; i < n_thr; ++i)
        if (!(thr[i] > thr[i - 1]))
            fail(XS_E_RUNTIME, "segment_volume: thresholds must be strictly increasing");
    if (n_class_map != n_thr + 1)
        fail(XS_E_RUNTIME, "segment_volume: class_map must cover all %d classes", n_thr + 1);
    if (n_thr > 15)
        fail(XS_E_UNSUPPORTED, "xscat-gpu: at most 16 segmentation classes supported");
}

static void check_density_phantom_args(const xs_class_spec* cls, int n_classes, const int32_t tgt[3],
                                       int n_materials)
{
    if (n_classes <= 0 || n_classes > 16)
        fail(XS_E_UNSUPPORTED, "xscat-gpu: 1..16 segmentation classes supported");
    if (tgt[0] <= 0 || tgt[1] <= 0 || tgt[2] <= 0)
        fail(XS_E_RUNTIME, "phantom: dims must be positive");
    if (n_materials <= 0)
        fail(XS_E_RUNTIME, "phantom: no material table");
    for (int l = 0; l < n_classes; ++l)
        if (cls[l].material_id < 0 || cls[l].material_id > 255)
            fail(XS_E_RUNTIME, "to_density_phantom: class material id out of range");
}

int xs_otsu_thresholds(xs_context* c, const float* volume, const int32_t dims[3], int32_t n_classes,
                       int32_t histogram_bins, double* thresholds, int32_t device_ptrs)
{
    return guard(c, [&] {
        const size_t nvox = (size_t)std::max(dims[0], 0) * std::max(dims[1], 0) * std::max(dims[2], 0);
        const float* vol = (n_classes >= 2 && n_classes <= 4 && histogram_bins >= n_classes && nvox)
                               ? seg_volume_in(c, volume, nvox, device_ptrs)
                               : volume;
        seg_otsu(c, vol, dims, n_classes, histogram_bins, thresholds);
    });
}

int xs_segment_volume(xs_context* c, const float* volume, uint64_t n_voxels, const double* thresholds,
                      int32_t n_thresholds, int32_t n_class_map, uint8_t* labels, int32_t device_ptrs)
{
    return guard(c, [&] {
        check_thresholds(thresholds, n_thresholds, n_class_map);
        if (!n_voxels)
            return;
        const float* vol = seg_volume_in(c, volume, n_voxels, device_ptrs);
        c->seg_thr.reserve(16);
        if (n_thresholds)
            cuda_check(cudaMemcpyAsync(c->seg_thr.p, thresholds, n_thresholds * sizeof(double),
                                       cudaMemcpyHostToDevice, c->stream),
                       "H2D");
        uint8_t* out = labels;
        if (!device_ptrs) {
            c->seg_labels.reserve(n_voxels);
            out = c->seg_labels.p;
        }
        cuda_check(xsd::launch_segment_labels(vol, n_voxels, c->seg_thr.p, n_thresholds, out, c->sm_count, c->stream),
                   "segment");
        if (!device_ptrs)
            cuda_check(cudaMemcpyAsync(labels, out, n_voxels, cudaMemcpyDeviceToHost, c->stream), "D2H");
        cuda_check(cudaStreamSynchronize(c->stream), "segment");
    });
}

// REF to_density_phantom's label check, then the phantom's validation
// (validate_phantom at recon.cpp:320) on the device outputs.
static void density_checks(xs_context* c, const uint8_t* labels_dev, const uint8_t* ids, const float* dens,
                           uint64_t n_out, int n_materials, const xs_material* materials)
{
    unsigned char ctl[64];
    cuda_check(cudaMemcpyAsync(ctl, c->seg_ctl.p, sizeof ctl, cudaMemcpyDeviceToHost, c->stream), "D2H");
    cuda_check(cudaStreamSynchronize(c->stream), "to_density_phantom");
    const unsigned long long bad = SegCtlView(ctl).first_bad();
    if (bad != ~0ull) {
        uint8_t l = 0;
        cuda_check(cudaMemcpy(&l, labels_dev + bad, 1, cudaMemcpyDeviceToHost), "D2H");
        fail(XS_E_RUNTIME, "to_density_phantom: unmapped label %d", (int)l);
    }
    if (!materials)
        return;
    xs_phantom ph{};
    ph.n_materials = n_materials;
    ph.materials = materials;
    std::vector<int> has_tables(n_materials, 0);
    uint32_t tab_bits = 0;
    for (int m = 1; m < n_materials && m < 32; ++m) {
        has_tables[m] = materials[m].mu.n > 0;
        tab_bits |= has_tables[m] ? (1u << m) : 0u;
    }
    cuda_check(xsd::launch_seg_reset(c->seg_ctl.p, c->stream), "validate");
    cuda_check(xsd::launch_phantom_scan(ids, dens, n_out, n_materials, tab_bits, c->seg_ctl.p, c->sm_count, c->stream),
               "validate");
    cuda_check(cudaMemcpyAsync(ctl, c->seg_ctl.p, sizeof ctl, cudaMemcpyDeviceToHost, c->stream), "D2H");
    cuda_check(cudaStreamSynchronize(c->stream), "validate");
    const unsigned long long vb = SegCtlView(ctl).first_bad();
    if (vb != ~0ull) {
        uint8_t id = 0;
        float d = 0.f;
        cuda_check(cudaMemcpy(&id, ids + vb, 1, cudaMemcpyDeviceToHost), "D2H");
        cuda_check(cudaMemcpy(&d, dens + vb, 4, cudaMemcpyDeviceToHost), "D2H");
        fail(XS_E_RUNTIME, "%s", voxel_error(ph, has_tables, id, d).c_str());
    }
}

int xs_to_density_phantom(xs_context* c, const uint8_t* labels, const int32_t src_dims[3],
                          const xs_class_spec* class_map, int32_t n_classes, const int32_t target_dims[3],
                          int32_t n_materials, const xs_material* materials, uint8_t* material_id, float* density,
                          int32_t device_ptrs)
{
    return guard(c, [&] {
        check_density_phantom_args(class_map, n_classes, target_dims, n_materials);
        const uint64_t n_src = (uint64_t)src_dims[0] * src_dims[1] * src_dims[2];
        const uint64_t n_out = (uint64_t)target_dims[0] * target_dims[1] * target_dims[2];
        const uint8_t* lab = labels;
        if (!device_ptrs) {
            c->seg_labels.reserve(n_src);
            cuda_check(cudaMemcpyAsync(c->seg_labels.p, labels, n_src, cudaMemcpyHostToDevice, c->stream), "H2D");
            lab = c->seg_labels.p;
        }
        uint8_t* ids = material_id;
        float* dens = density;
        if (!device_ptrs) {
            c->seg_ids.reserve(n_out);
            c->seg_dens.reserve(n_out);
            ids = c->seg_ids.p;
            dens = c->seg_dens.p;
        }
        int mat[16];
        double rho[16];
        for (int l = 0; l < n_classes; ++l) {
            mat[l] = class_map[l].material_id;
            rho[l] = class_map[l].density;
        }
        const int s3[3] = {src_dims[0], src_dims[1], src_dims[2]}, t3[3] = {target_dims[0], target_dims[1], target_dims[2]};
        c->seg_ctl.reserve(xsd::seg_ctl_bytes());
        cuda_check(xsd::launch_seg_reset(c->seg_ctl.p, c->stream), "to_density_phantom");
        cuda_check(xsd::launch_density_phantom(lab, nullptr, s3, t3, mat, rho, n_classes, nullptr, 0, ids, dens,
                                               c->seg_ctl.p, c->sm_count, c->stream),
                   "to_density_phantom");
        density_checks(c, lab, ids, dens, n_out, n_materials, materials);
        if (!device_ptrs) {
            cuda_check(cudaMemcpyAsync(material_id, ids, n_out, cudaMemcpyDeviceToHost, c->stream), "D2H");
            cuda_check(cudaMemcpyAsync(density, dens, n_out * 4, cudaMemcpyDeviceToHost, c->stream), "D2H");
            cuda_check(cudaStreamSynchronize(c->stream), "D2H");
        }
    });
}

int xs_segment_to_scene(xs_context* c, const float* volume, const int32_t dims[3], const double voxel_size[3],
                        int32_t n_classes, int32_t histogram_bins, const xs_class_spec* class_map,
                        const int32_t target_dims[3], int32_t n_materials, const xs_material* materials,
                        double* thresholds, int32_t device_ptrs)
{
    return guard(c, [&] {
        const size_t nvox = (size_t)std::max(dims[0], 0) * std::max(dims[1], 0) * std::max(dims[2], 0);
        const float* vol = (n_classes >= 2 && n_classes <= 4 && histogram_bins >= n_classes && nvox)
                               ? seg_volume_in(c, volume, nvox, device_ptrs)
                               : volume;
        // REF correction.cpp:168-171: otsu -> segment_volume -> to_density_phantom
        seg_otsu(c, vol, dims, n_classes, histogram_bins, thresholds);
        check_thresholds(thresholds, n_classes - 1, n_classes);
        check_density_phantom_args(class_map, n_classes, target_dims, n_materials);
        const uint64_t n_out = (uint64_t)target_dims[0] * target_dims[1] * target_dims[2];
        c->seg_ids.reserve(n_out);
        c->seg_dens.reserve(n_out);
        int mat[16];
        double rho[16];
        for (int l = 0; l < n_classes; ++l) {
            mat[l] = class_map[l].material_id;
            rho[l] = class_map[l].density;
        }
        const int s3[3] = {dims[0], dims[1], dims[2]}, t3[3] = {target_dims[0], target_dims[1], target_dims[2]};
        cuda_check(xsd::launch_seg_reset(c->seg_ctl.p, c->stream), "segmentation");
        cuda_check(xsd::launch_density_phantom(nullptr, vol, s3, t3, mat, rho, n_classes, thresholds, n_classes - 1,
                                               c->seg_ids.p, c->seg_dens.p, c->seg_ctl.p, c->sm_count, c->stream),
                   "segmentation");
        // REF to_density_phantom: voxel size = vol voxel * dims / target, centred grid
        xs_phantom ph{};
        for (int a = 0; a < 3; ++a) {
            ph.dims[a] = target_dims[a];
            ph.voxel_size[a] = voxel_size[a] * dims[a] / target_dims[a];
            ph.origin[a] = (-target_dims[a] * ph.voxel_size[a]) * 0.5;
        }
        ph.material_id = c->seg_ids.p;
        ph.density = c->seg_dens.p;
        ph.n_materials = n_materials;
        ph.materials = materials;
        upload_phantom_impl(c, &ph, true);
        if (const char* dir = std::getenv("XSCAT_DUMP_SCENE")) { // diagnostics: the segmented ids
            static int k = 0;
            std::vector<uint8_t> ids(n_out);
            cuda_check(cudaMemcpy(ids.data(), c->seg_ids.p, n_out, cudaMemcpyDeviceToHost), "dump");
            const std::string path = std::string(dir) + "/scene_" + std::to_string(k++) + ".u8";
            if (FILE* f = std::fopen(path.c_str(), "wb")) {
                std::fwrite(ids.data(), 1, n_out, f);
                std::fclose(f);
            }
        }
    });
}

// ------------------------------------------------ iterative correction
// REF run_iterative_correction (correction.cpp:137-266) with every stage on
// the device: ln conversion, FDK, segmentation -> scene, scatter and primary
// scans, the fused post-processing + Eq. 8 tail, FDK of the corrected stack.
// Only thresholds, statistics and the reports cross to the host.
void xs_correction_config_default(xs_correction_config* cc)
{
    std::memset(cc, 0, sizeof *cc);
    cc->n_iterations = 3;
    cc->simulate_every_kth_angle = 2;
    cc->recon_dims[0] = cc->recon_dims[1] = cc->recon_dims[2] = 64;
    cc->n_classes = 3;
    xs_sim_config_default(&cc->sim);
    cc->sg_window = 15;
    cc->sg_polyorder = 3;
    cc->sg_auto_window = 1;
}

// The loop's scans: on this context, or sharded by angle over a group's
// devices when a group installed its delegate (xs_group_run_iterative_correction).
static void loop_scan(xs_context* c, const xs_geometry* g, const xs_spectrum* spec, const xs_sim_config* cfg,
                      const int32_t* subset, int32_t n, int32_t what, double* d_primary, double* d_scatter)
{
    if (c->scan_hook)
        c->scan_hook(g, spec, cfg, subset, n, what, d_primary, d_scatter);
    else
        scan_device_impl(c, g, spec, cfg, subset, n, what, d_primary, d_scatter, nullptr);
}

static void call_status(xs_context* c, int st)
{
    if (st != XS_OK)
        fail(st, "%s", c->err.c_str());
}

static void loop_stage(xs_context* c, int iteration, const char* name, const std::function<void()>& f)
{
    const xsi::Range range(name);
    try {
        f();
    } catch (const Error& e) { // REF correction.cpp:22-31
        fail(XS_E_RUNTIME, "iteration %d, stage %s: %s", iteration, name, e.msg.c_str());
    }
    (void)c;
}

int xs_run_iterative_correction(xs_context* c, const double* raw_intensity, const double* flatfield,
                                const xs_geometry* g, const xs_spectrum* spec, const xs_correction_config* cc,
                                int32_t n_materials, const xs_material* materials, float* corrected_volume,
                                double* corrected_stack, xs_iteration_report* reports, int32_t device_ptrs)
{
    return guard(c, [&] {
        using clk = std::chrono::steady_clock;
        auto secs = [](clk::time_point t0) { return std::chrono::duration<double>(clk::now() - t0).count(); };
        // REF validate_correction_config (correction.cpp:35-59), n_materials incl. vacuum
        if (cc->n_iterations < 1)
            fail(XS_E_RUNTIME, "correction config: n_iterations must be >= 1");
        if (cc->simulate_every_kth_angle < 1)
            fail(XS_E_RUNTIME, "correction config: simulate_every_kth_angle must be >= 1");
        if (cc->n_classes < 2 || cc->n_classes > 4)
            fail(XS_E_RUNTIME, "correction config: n_classes must be in [2,4]");
        if (!cc->class_map)
            fail(XS_E_RUNTIME, "correction config: class_map must have n_classes entries");
        for (int l = 0; l < cc->n_classes; ++l) {
            const xs_class_spec& k = cc->class_map[l];
            if (k.material_id < 0 || k.material_id >= n_materials)
                fail(XS_E_RUNTIME, "correction config: class material id %d out of range", k.material_id);
            if (k.material_id == 0 && k.density != 0.0)
                fail(XS_E_RUNTIME, "correction config: vacuum class must have density 0");
            if (k.density < 0.0)
                fail(XS_E_RUNTIME, "correction config: negative class density");
        }
        for (int d : cc->recon_dims)
            if (d <= 0)
                fail(XS_E_RUNTIME, "correction config: recon dims must be positive");
        xsh::validate_sim_config(cc->sim);
        xsh::validate_geometry(*g);
        if (!c->have_response)
            fail(XS_E_RUNTIME, "xscat-gpu: no detector response uploaded (xs_upload_response)");
        const int nu = g->nu, nv = g->nv, n_full = g->n_angles;
        const int mc_nu = cc->mc_nu > 0 ? cc->mc_nu : nu, mc_nv = cc->mc_nv > 0 ? cc->mc_nv : nv;
        if ((long long)mc_nv * nu != (long long)mc_nu * nv)
            fail(XS_E_RUNTIME, "run_iterative_correction: mc grid must preserve the detector aspect ratio");
        xs_geometry g_mc = *g;
        g_mc.nu = mc_nu;
        g_mc.nv = mc_nv;
        g_mc.pixel_pitch = g->pixel_pitch * g->nu / mc_nu;
        int32_t sg_w = cc->sg_window, sg_o = cc->sg_polyorder;
        if (cc->sg_auto_window) {
            int32_t dummy;
            xs_default_sg_spec(mc_nu, mc_nv, &sg_w, &dummy);
        }
        if (xs_validate_sg_spec(sg_w, sg_o) != XS_OK)
            fail(XS_E_RUNTIME, "%s", xs_last_error(nullptr));
        std::vector<int32_t> sub, all(n_full);
        for (int i = 0; i < n_full; i += cc->simulate_every_kth_angle)
            sub.push_back(i);
        std::vector<double> sub_angles;
        for (int i : sub)
            sub_angles.push_back(g->angles[i]);
        for (int i = 0; i < n_full; ++i)
            all[i] = i;
        const size_t np = (size_t)nu * nv, np_mc = (size_t)mc_nu * mc_nv;
        const size_t nvox = (size_t)cc->recon_dims[0] * cc->recon_dims[1] * cc->recon_dims[2];
        cudaStream_t st = c->stream;

        // One-time path (REF :171-178): a = ln(flat / I), FDK of a
        c->loop_a.reserve(np * n_full);
        c->loop_c.reserve(np * n_full);
        const double* raw = raw_intensity;
        const double* flat = flatfield;
        if (!device_ptrs) {
            cuda_check(cudaMemcpyAsync(c->loop_c.p, raw_intensity, np * n_full * 8, cudaMemcpyHostToDevice, st), "H2D");
            c->loop_flat.reserve(np);
            cuda_check(cudaMemcpyAsync(c->loop_flat.p, flatfield, np * 8, cudaMemcpyHostToDevice, st), "H2D");
            raw = c->loop_c.p;
            flat = c->loop_flat.p;
        }
        call_status(c, xs_intensity_to_attenuation(c, raw, flat, nu, nv, n_full, c->loop_a.p, 1));
        double voxel[3];
        xs_default_voxel_size(g, cc->recon_dims, voxel);
        c->loop_vol[0].reserve(nvox);
        c->loop_vol[1].reserve(nvox);
        call_status(c, xs_fbp_reconstruct(c, c->loop_a.p, g->angles, n_full, nu, nv, g, cc->recon_dims, voxel, 1,
                                          c->loop_vol[0].p, 1));
        c->loop_scat.reserve(np_mc * sub.size());
        c->loop_prim.reserve(np_mc * n_full);
        c->loop_ncc.reserve(xsd::ncc_scratch_bytes() / 8);
        int prev = 0;
        for (int iter = 1; iter <= cc->n_iterations; ++iter) {
            xs_iteration_report rep{};
            rep.iteration = iter;
            const auto t_iter = clk::now();
            auto t0 = clk::now();
            double thr[4];
            loop_stage(c, iter, "segmentation", [&] {
                call_status(c, xs_segment_to_scene(c, c->loop_vol[prev].p, cc->recon_dims, voxel, cc->n_classes, 1024,
                                                   cc->class_map, cc->recon_dims, n_materials, materials, thr, 1));
            });
            rep.seconds_segmentation = secs(t0);
            t0 = clk::now();
            loop_stage(c, iter, "mc-scatter", [&] {
                loop_scan(c, &g_mc, spec, &cc->sim, sub.data(), (int32_t)sub.size(), 1, nullptr, c->loop_scat.p);
            });
            rep.seconds_mc_scatter = secs(t0);
            t0 = clk::now();
            loop_stage(c, iter, "mc-primary", [&] {
                loop_scan(c, &g_mc, spec, &cc->sim, all.data(), n_full, 0, c->loop_prim.p, nullptr);
            });
            rep.seconds_mc_primary = secs(t0);
            rep.mc_seconds_per_projection = rep.seconds_mc_scatter / (double)sub.size();
            // REF :199-246 post-processing, scatter fraction and Eq. 8, fused
            t0 = clk::now();
            uint64_t clamped = 0;
            loop_stage(c, iter, "postprocess", [&] {
                call_status(c, xs_correction_tail(c, c->loop_scat.p, sub_angles.data(), (int32_t)sub.size(),
                                                  c->loop_prim.p, g->angles, n_full, mc_nu, mc_nv, sg_w, sg_o,
                                                  c->loop_a.p, nu, nv, c->loop_c.p, &rep.mean_scatter_fraction,
                                                  &clamped, 1));
            });
            rep.seconds_postprocess = secs(t0);
            rep.seconds_correction = 0.0; // fused into the tail above
            rep.negative_scatter_clamped = clamped;
            t0 = clk::now();
            loop_stage(c, iter, "fbp", [&] {
                call_status(c, xs_fbp_reconstruct(c, c->loop_c.p, g->angles, n_full, nu, nv, g, cc->recon_dims, voxel,
                                                  1, c->loop_vol[prev ^ 1].p, 1));
            });
            rep.seconds_fbp = secs(t0);
            // REF :255-256 ncc(corrected, previous)
            double m[5];
            cuda_check(xsd::launch_ncc(c->loop_vol[prev ^ 1].p, c->loop_vol[prev].p, nvox, c->loop_ncc.p, st), "ncc");
            cuda_check(cudaMemcpyAsync(m, c->loop_ncc.p, sizeof m, cudaMemcpyDeviceToHost, st), "D2H");
            cuda_check(cudaStreamSynchronize(st), "ncc");
            if (!(m[3] > 0.0) || !(m[4] > 0.0))
                fail(XS_E_RUNTIME, "ncc: zero variance input");
            rep.ncc_to_previous = m[2] / std::sqrt(m[3] * m[4]);
            prev ^= 1;
            rep.seconds_total = secs(t_iter);
            if (reports)
                reports[iter - 1] = rep;
        }
        const cudaMemcpyKind k = device_ptrs ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
        if (corrected_volume)
            cuda_check(cudaMemcpyAsync(corrected_volume, c->loop_vol[prev].p, nvox * 4, k, st), "volume out");
        if (corrected_stack)
            cuda_check(cudaMemcpyAsync(corrected_stack, c->loop_c.p, np * n_full * 8, k, st), "stack out");
        cuda_check(cudaStreamSynchronize(st), "run_iterative_correction");
    });
}

} // extern "C"

// ================================================ internal API (multi.cu)
namespace xsi {

int run(xs_context* c, const std::function<void()>& f)
{
    return guard(c, f);
}

int device(const xs_context* c) { return c->device; }
cudaStream_t stream(const xs_context* c) { return c->stream; }
void*& mgpu_slot(xs_context* c) { return c->mgpu; }
void set_scan_hook(xs_context* c, ScanHook h) { c->scan_hook = std::move(h); }

uint64_t history_count(const xs_geometry& g, const xs_spectrum& spec, const xs_sim_config& cfg)
{
    return make_plan(g, spec, cfg).n_hist;
}

xs_accum_layout layout(const xs_geometry& g, const xs_spectrum& spec, const xs_sim_config& cfg)
{
    return make_plan(g, spec, cfg).layout;
}

unsigned long long* own_accum(xs_context* c, size_t words)
{
    c->accum.reserve(words);
    return c->accum.p;
}

void accumulate(xs_context* c, const xs_geometry& g, int angle, const xs_spectrum& spec, const xs_sim_config& cfg,
                uint64_t h0, uint64_t h1, unsigned long long* d_accum)
{
    validate_call(g, angle, spec, cfg, "simulate_scatter");
    ::accumulate(c, g, angle, spec, cfg, h0, h1, d_accum);
}

void finalize(xs_context* c, const xs_geometry& g, const xs_spectrum& spec, const xs_sim_config& cfg,
              const unsigned long long* const* srcs, int n_src, uint64_t h0, uint64_t h1, xs_scatter_result* out,
              double* d_image)
{
    ::finalize(c, g, spec, cfg, srcs, n_src, h0, h1, out, d_image);
}

void scan_device(xs_context* c, const xs_geometry* g, const xs_spectrum* spec, const xs_sim_config* cfg,
                 const int32_t* subset, int32_t n, int32_t what, double* d_primary, double* d_scatter,
                 double* seconds)
{
    scan_device_impl(c, g, spec, cfg, subset, n, what, d_primary, d_scatter, seconds);
}

void check_scan_args(const xs_geometry* g, const xs_sim_config* cfg, const int32_t* subset, int32_t n)
{
    if (n <= 0)
        fail(XS_E_RUNTIME, "run_scan: empty angle subset");
    xsh::validate_sim_config(*cfg);
    xsh::validate_geometry(*g);
    for (int i = 0; i < n; ++i)
        if (subset[i] < 0 || subset[i] >= g->n_angles)
            fail(XS_E_OUT_OF_RANGE, "run_scan: angle index %d out of range", subset[i]);
}

void cuda(cudaError_t e, const char* what) { cuda_check(e, what); }

} // namespace xsi
